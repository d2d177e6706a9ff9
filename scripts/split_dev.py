"""Development timing of the two-kernel head (head_split.cu) on one GPU,
Llama shape, |I| = 3072, n = 60, k = 10: head calls in a CUDA graph over R
rotating active sets (cold L2) and over one set (warm), the fused step, and a
phase trace of kernels A and B.  Experiment flags: NANOSPEC_SPLIT_FLAGS
(1 = skip kernel B, 2 = no PDL).

    python scripts/split_dev.py [--mode 7] [--trace]
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
ap.add_argument("--mode", type=int, default=-1)
ap.add_argument("--trace", action="store_true")
ap.add_argument("--n", type=int, default=60)
ap.add_argument("--R", type=int, default=24)
args = ap.parse_args()
dev = torch.device("cuda", 0)
V, d, n, k, Wm = 128256, 4096, args.n, 10, 3072
if args.mode != -1:
    N.check(N.lib().nanospec_debug_set_head_mode(args.mode), "mode")
W = SI.bf16_weights(V, d, seed=0, device=dev)
R = args.R
pools = SI.disjoint_pools(V, Wm + 126, R, seed=3)
states, outs, ud, uv = [], [], [], []
Hs = SI.bf16_hidden(n, d, seed=1, device=dev, batch=R)
for r in range(R):
    prompt, ups = SI.cyclic_fresh_updates(pools[r], Wm, 40)
    st = P.ActiveVocab(V, Wm, device=dev)
    st.init(0, torch.as_tensor(prompt, device=dev))
    states.append(st)
    outs.append(P.HeadOutputs(1, n, k, Wm, dev))
    ud.append(torch.as_tensor(np.stack([u[0] for u in ups]), device=dev))
    uv.append(torch.as_tensor(np.stack([u[1] for u in ups]), device=dev))
torch.cuda.synchronize()
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def graph_time(fn, count, reps=5):
    for s in range(3):
        fn(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for s in range(count):
            fn(s)
    ts = []
    for _ in range(reps):
        e0.record(stream)
        g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / count)
    return float(np.median(ts))


cur = [5] * R


def head_cold(s):
    r = s % R
    P.draft_logits_topk(states[r], W, Hs[r:r + 1], k, out=outs[r])


def head_warm(s):
    P.draft_logits_topk(states[0], W, Hs[0:1], k, out=outs[0])


def step_cold(s):
    r = s % R
    c = cur[r] % 40
    cur[r] += 1
    P.step(states[r], 0, ud[r][c], uv[r][c], W, Hs[r], k, out=outs[r])


tag = f"mode {args.mode} flags {os.environ.get('NANOSPEC_SPLIT_FLAGS', '0')} n {n}"
print(f"{tag}: head cold {graph_time(head_cold, 48):.2f} us, warm {graph_time(head_warm, 48):.2f} us")
if os.environ.get("NANOSPEC_SPLIT_FLAGS", "0") == "0":
    print(f"{tag}: fused step cold {graph_time(step_cold, 24, reps=1):.2f} us")

if args.trace:
    trace = torch.zeros(1024 * 16, dtype=torch.int64, device=dev)
    for it in range(2):
        torch.cuda.synchronize()
        N.check(N.lib().nanospec_debug_set_trace(trace.data_ptr(), 1024), "trace")
        trace.zero_()
        fn = head_cold if it == 0 else (lambda s: step_cold(s))
        fn(7)
        torch.cuda.synchronize()
        N.check(N.lib().nanospec_debug_set_trace(None, 0), "trace")
        t = trace.view(1024, 16).cpu().numpy().astype(np.int64)
        live = t[:, 0] > 0
        t0 = t[live, 0].min()
        rows = np.nonzero(live)[0]
        # A rows are a contiguous block from 0; B rows follow
        nA = int(np.argmax(t[:, 12] == 0xB)) if (t[:, 12] == 0xB).any() else int(live.sum())
        print(f"trace {'head' if it == 0 else 'fused step'}: A CTAs {nA}, B CTAs {len(rows) - nA}")
        if nA > 147 and t[nA - 1, 10] > 0:  # the fused step's updater (last stream CTA): its phases
            u = t[nA - 1]
            print("    updater: " + ", ".join(f"{nm} {(u[e] - t0) / 1e3:.2f}" for nm, e in
                                           (("start", 0), ("dep", 1), ("lists", 10), ("ring", 11), ("counts", 12),
                                            ("written", 14), ("exit", 9)) if u[e] > 0))
        for name, e in (("A start", 0), ("A dep", 1), ("A ids", 7), ("A first loads", 2), ("A loads landed", 3), ("A last MMA", 4),
                        ("A drained", 9), ("upd published", 11)):
            c = t[:nA, e]
            c = c[c > 0]
            if len(c):
                r_ = (c - t0) / 1e3
                print(f"    {name:16s} n={len(c):3d} min {r_.min():6.2f} med {np.median(r_):6.2f} max {r_.max():6.2f}")
        cy = t[:nA, 13] - t[:nA, 12]
        print("    A cycles ids->first loads:", np.percentile(cy[(t[:nA, 13] > 0)], [0, 50, 100]))
        for nm, rows_ in (("A", t[:nA]), ("B", t[nA:nA + 512][t[nA:nA + 512, 12] == 0xB])):
            ok = (rows_[:, 15] > 0) & (rows_[:, 14] > 0)
            if ok.any():
                cyc = rows_[ok, 15] - rows_[ok, 14]
                ns = rows_[ok, 9 if nm == "A" else 4] - rows_[ok, 0 if nm == "A" else 1]
                print(f"    {nm} SM clock ~{np.median(cyc / np.maximum(ns, 1)) * 1e3:.0f} MHz")
        Bt = t[nA:nA + 512][t[nA:nA + 512, 12] == 0xB]
        if len(Bt):
            print("    B merge cycles: threshold", np.median(Bt[:, 8]), "staged", np.median(Bt[:, 10]),
                  "cands", np.median(Bt[:, 11]), "ranked+stored", np.median(Bt[:, 13]))
        for name, e in (("B start", 0), ("B dep", 1), ("B loaded", 5), ("B hist1", 6), ("B S1", 2), ("B cands", 7), ("B ranked", 9), ("B tiles", 3), ("B done", 4)):
            c = t[nA:nA + 512, e]
            c = c[c > 0]
            if len(c):
                r_ = (c - t0) / 1e3
                print(f"    {name:16s} n={len(c):3d} min {r_.min():6.2f} med {np.median(r_):6.2f} max {r_.max():6.2f}")

if args.trace:
    # three consecutive steps (head-only, then fused) captured in ONE graph, each
    # with its own trace region: the overlap / gaps between consecutive launches
    for what in ("head", "step"):
        regs = [torch.zeros(1024 * 16, dtype=torch.int64, device=dev) for _ in range(3)]
        fn = head_cold if what == "head" else step_cold
        for s in range(3):
            fn(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for s in range(3):
                N.check(N.lib().nanospec_debug_set_trace(regs[s].data_ptr(), 1024), "trace")
                fn(10 + s)
        N.check(N.lib().nanospec_debug_set_trace(None, 0), "trace")
        g.replay()
        torch.cuda.synchronize()
        ts = [r.view(1024, 16).cpu().numpy().astype(np.int64) for r in regs]
        t0 = min(t[t[:, 0] > 0, 0].min() for t in ts)
        print(f"graph of 3 {what} calls (us from the first stream CTA start):")
        for s, t in enumerate(ts):
            nA = int(np.argmax(t[:, 12] == 0xB)) if (t[:, 12] == 0xB).any() else int((t[:, 0] > 0).sum())
            A, B = t[:nA], t[nA:nA + 512]
            B = B[B[:, 12] == 0xB]
            def rng(c):
                c = c[c > 0]
                return f"{(c.min() - t0) / 1e3:6.2f}..{(c.max() - t0) / 1e3:6.2f}" if len(c) else "-"
            print(f"  call {s}: A start {rng(A[:, 0])} dep {rng(A[:, 1])} first loads {rng(A[:, 2])} "
                  f"drained {rng(A[:, 9])} | B start {rng(B[:, 0])} dep {rng(B[:, 1])} done {rng(B[:, 4])}")
