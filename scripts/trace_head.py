"""Phase timeline of one fused head call (debug trace, globaltimer ns per CTA).

    python scripts/trace_head.py [--n 60] [--m 3072] [--cold]
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_26444_b200 as P  # noqa: E402
from paper_2605_26444_b200 import _native as N  # noqa: E402
from synthetic import inputs as SI  # noqa: E402

EVENTS = ["start", "dep_ok", "rowptr", "loads_landed", "mma_done", "fin_go", "-", "ids_ready",
          "done", "drained", "l1|fin_staged", "l2|fin_summed|upd_done|stage0_full", "l2staged|pub_seen|stage_mid_full",
          "l1_all|upd_counts|stage_last_full"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=60)
    ap.add_argument("--m", type=int, default=3072)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--step", action="store_true", help="trace the fused step (update + head) instead")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    V, d = 128256, 4096
    W = SI.bf16_weights(V, d, seed=0, device=dev)
    ids = np.random.default_rng(0).choice(V, args.m, replace=False).astype(np.int32)
    st = P.ActiveVocab(V, 3072 if args.m <= 3072 else args.m, device=dev)
    if args.step:  # headline recipe: |I| = W_max, 63 fresh ids per step
        pool = SI.disjoint_pools(V, st.w_max + 126, 1, seed=5)[0]
        ids, ups = SI.cyclic_fresh_updates(pool, st.w_max, 4 * args.reps + 4)
        upd_iter = iter([(torch.as_tensor(a, device=dev), torch.as_tensor(b, device=dev)) for a, b in ups])
    st.init(0, torch.as_tensor(ids, device=dev))
    H = SI.bf16_hidden(args.n, d, seed=1, device=dev).reshape(1, args.n, d)
    out = P.HeadOutputs(1, args.n, args.k, st.w_max, dev)
    trace = torch.zeros(256 * 16 + 512, dtype=torch.int64, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        P.draft_logits_topk(st, W, H, args.k, impl="tc", out=out)
    torch.cuda.synchronize()
    for mode in ("cold", "warm"):
        rows = []
        for r in range(args.reps):
            if mode == "cold":
                flush.fill_(r & 0xff)
            torch.cuda.synchronize()
            trace.zero_()
            N.check(N.lib().nanospec_debug_set_trace(trace.data_ptr(), 256), "set_trace")
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if args.step:
                dd, vv = next(upd_iter)
                P.step(st, 0, dd, vv, W, H[0], args.k, out=out)
            else:
                P.draft_logits_topk(st, W, H, args.k, impl="tc", out=out)
            e1.record()
            torch.cuda.synchronize()
            N.check(N.lib().nanospec_debug_set_trace(None, 0), "set_trace")
            full = trace.cpu().numpy().astype(np.int64)
            clk = full[256 * 16:].reshape(256, 2)
            t = full[:256 * 16].reshape(256, 16)
            ctas = int((t[:, 0] > 0).sum())
            t = t[:ctas]
            t0 = t[:, 0].min()
            rows.append((e0.elapsed_time(e1) * 1e3, t, t0))
        print(f"=== {mode} (m={args.m}, n={args.n}); event-timed call: "
              f"{np.median([r[0] for r in rows]):.2f} us median of {args.reps}")
        ev_us, t, t0 = rows[-1]
        cyc = t[:, 15] - t[:, 14]
        ns = t[:, 8] - t[:, 0]
        ok = (t[:, 15] > 0) & (ns > 0)
        if ok.any():
            print(f"  SM clock during the call: {np.median(cyc[ok] / ns[ok]):.3f} GHz (median over CTAs)")
        t[:, 14:16] = 0

        for e, name in enumerate(EVENTS):
            col = t[:, e]
            col = col[col > 0]
            if len(col) == 0:
                continue
            rel = (col - t0) / 1e3
            print(f"  {name:13s} n={len(col):3d}  min {rel.min():7.2f}  med {np.median(rel):7.2f}  max {rel.max():7.2f} us")
        if args.step and t.shape[0] > 125:  # fused: the patch cluster (CTAs 120-124) and the update cluster
            for b0, label in ((120, "patch"), (125, "update")):
                sel = t[b0:b0 + 5]
                vals = {name: (sel[:, e][sel[:, e] > 0] - t0).max() / 1e3 for e, name in enumerate(EVENTS)
                        if (sel[:, e] > 0).any()}
                print(f"  {label} cluster (max over its CTAs):", {k: round(v, 2) for k, v in vals.items()})


def trace_state():
    dev = torch.device("cuda", 0)
    V = 128256
    pools = SI.disjoint_pools(V, 3072 + 126, 1)
    prompt, ups = SI.cyclic_fresh_updates(pools[0], 3072, 8)
    st = P.ActiveVocab(V, 3072, device=dev)
    st.init(0, torch.as_tensor(prompt, device=dev))
    trace = torch.zeros(256 * 16, dtype=torch.int64, device=dev)
    names = ["start", "staged", "ring_read", "counts", "-", "done"]
    for i, (d, v) in enumerate(ups):
        dd, vv = torch.as_tensor(d, device=dev), torch.as_tensor(v, device=dev)
        torch.cuda.synchronize()
        N.check(N.lib().nanospec_debug_set_trace(trace.data_ptr(), 256), "set_trace")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st.update(0, dd, vv)
        e1.record()
        torch.cuda.synchronize()
        N.check(N.lib().nanospec_debug_set_trace(None, 0), "set_trace")
        t = trace.view(256, 16)[0].cpu().numpy().astype(np.int64)
        rel = [(t[9 + j] - t[9]) / 1e3 for j in range(6)]
        print(f"state update {i}: event {e0.elapsed_time(e1) * 1e3:.2f} us; " +
              " ".join(f"{n}={r:.2f}" for n, r in zip(names, rel)))


if __name__ == "__main__":
    if "--state" in sys.argv:
        sys.argv.remove("--state")
        trace_state()
    main()
