"""Event-timed head calls (no trace) for the pair kernel under NANOSPEC_PAIR_DBG."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_26444_b200 as P  # noqa: E402
from paper_2605_26444_b200 import _native as N  # noqa: E402
from synthetic import inputs as SI  # noqa: E402

dev = torch.device("cuda", 0)
V, d, n, k = 128256, 4096, 60, 10
N.check(N.lib().nanospec_debug_set_head_mode(int(os.environ.get("MODE", "6"))), "mode")
W = SI.bf16_weights(V, d, seed=0, device=dev)
ids = np.random.default_rng(0).choice(V, 3072, replace=False).astype(np.int32)
st = P.ActiveVocab(V, 3072, device=dev)
st.init(0, torch.as_tensor(ids, device=dev))
H = SI.bf16_hidden(n, d, seed=1, device=dev).reshape(1, n, d)
out = P.HeadOutputs(1, n, k, 3072, dev)
for _ in range(5):
    P.draft_logits_topk(st, W, H, k, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    P.draft_logits_topk(st, W, H, k, out=out)
e1.record()
torch.cuda.synchronize()
print(f"DBG {os.environ.get('NANOSPEC_PAIR_DBG', '0')} MODE {os.environ.get('MODE', '6')}: "
      f"{e0.elapsed_time(e1) * 1e3 / 50:.2f} us per head call (warm, back to back)")
