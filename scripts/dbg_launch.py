import torch, sys
sys.path.insert(0, '/root/repo')
import paper_2605_26444_b200 as P
from paper_2605_26444_b200 import _native as N
from synthetic import inputs as SI
import ctypes
V, d = 128256, 4096
W = SI.bf16_weights(V, d, seed=0, device="cuda")
H = SI.bf16_hidden(4, d, seed=2, device="cuda")
ids = torch.arange(V, dtype=torch.int32, device="cuda")
nid = torch.tensor([V], dtype=torch.int32, device="cuda")
try:
    P.logits_topk_ids(ids, nid, W, H, 10, debug_logits=True, impl="tc")
except Exception as e:
    print("call failed:", e)
try:
    torch.cuda.synchronize(); print("sync ok")
except Exception as e:
    print("sync:", e)
