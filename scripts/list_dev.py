"""Development timing + phase trace of the list mode (persistent split-K 1):
dp64-shaped batched head (B sequences, |I| = 3072, n = 60, k = 10) and the
dense [0, V) head.  Per CTA: last MMA commit, the epilogue's last unit start /
end and its total busy time.

    python scripts/list_dev.py [--B 64]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_26444_b200 as P  # noqa: E402
from paper_2605_26444_b200 import _native as N  # noqa: E402
from synthetic import inputs as SI  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=64)
args = ap.parse_args()
dev = torch.device("cuda", 0)
V, d, n, k, Wm, B = 128256, 4096, 60, 10, 3072, args.B
W = SI.bf16_weights(V, d, seed=0, device=dev)
pools = SI.disjoint_pools(V, Wm + 126, 40, seed=3)
st = P.ActiveVocab(V, Wm, device=dev, batch=B)
for b in range(B):
    prompt, _ = SI.cyclic_fresh_updates(pools[b % 40], Wm, 1)
    st.init(b, torch.as_tensor(prompt, device=dev))
H = SI.bf16_hidden(n, d, seed=1, device=dev, batch=B)
out = P.HeadOutputs(B, n, k, Wm, dev)
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def run():
    P.draft_logits_topk(st, W, H, k, out=out)


for _ in range(3):
    run()
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0.record(stream)
    run()
    e1.record(stream)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print(f"B={B}: head {np.median(ts):.1f} us (min {min(ts):.1f})")
NT = 8192
trace = torch.zeros(NT * 16, dtype=torch.int64, device=dev)
N.check(N.lib().nanospec_debug_set_trace(trace.data_ptr(), NT), "trace")
run()
torch.cuda.synchronize()
N.check(N.lib().nanospec_debug_set_trace(None, 0), "trace")
t = trace.view(NT, 16).cpu().numpy().astype(np.int64)
nA = 148
A = t[:nA]
t0 = A[A[:, 0] > 0, 0].min()
for name, e in (("A start", 0), ("A dep", 1), ("A first loads", 2), ("A last MMA commit", 4), ("E last unit start", 5),
                ("E last unit end", 6), ("A exit", 9)):
    c = A[:, e]
    c = c[c > 0]
    if len(c):
        r_ = (c - t0) / 1e3
        print(f"    {name:20s} n={len(c):3d} min {r_.min():8.2f} med {np.median(r_):8.2f} max {r_.max():8.2f}")
print("    tail item 0 cycles: kth", np.median(A[:, 10]), "compact", np.median(A[:, 11]), "cnt", np.median(A[:, 12]), "ranked", np.median(A[:, 13]))
Bm = t[nA:][t[nA:, 12] == 0xB]
for name, e in (("M start", 0), ("M dep", 1), ("M heads", 5), ("M cands", 7), ("M done", 4)):
    c = Bm[:, e]
    c = c[c > 0]
    if len(c):
        r_ = (c - t0) / 1e3
        print(f"    {name:20s} n={len(c):4d} min {r_.min():8.2f} med {np.median(r_):8.2f} max {r_.max():8.2f}")
busy = A[:, 8] / 1e3
units = A[:, 10] + 1
print(f"    epilogue busy per unit (us): med {np.median(busy / np.maximum(units, 1)):.2f} max {np.max(busy / np.maximum(units, 1)):.2f}; units per CTA {np.bincount(units)}")
