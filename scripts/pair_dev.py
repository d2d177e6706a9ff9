"""Development check of the pair-split head (head_pair.cu) on one GPU: forced
mode 6, Llama shape; logits vs a torch fp32 reference, top-k / lse, the fused
step vs update + head, and a phase trace.

    python scripts/pair_dev.py [--n 60] [--m 3072] [--k 10]
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

EV = ["start", "ids", "issued", "acc", "paired", "level1", "barrier", "level2"]


def ref_check(W, H, ids, v, i, l, z, k, tag):
    Wg = W[torch.as_tensor(ids, device=W.device).long()].float()
    zr = (H.float() @ Wg.T)  # [n, m]
    A = (H.float().abs() @ Wg.abs().T)
    if z is not None:
        err = (z[:, : len(ids)] - zr).abs() / torch.maximum(zr.abs(), A / 64)
        print(f"  [{tag}] logits max rel err {err.max().item():.2e}")
    tv, ti = torch.topk(zr, min(k, len(ids)), dim=1)
    gid = torch.as_tensor(ids, device=W.device)[ti]
    ok_v = torch.allclose(v[:, : tv.shape[1]], tv, rtol=2e-3, atol=1e-3)
    same = (i[:, : tv.shape[1]] == gid).float().mean().item()
    lr = torch.logsumexp(zr, dim=1)
    print(f"  [{tag}] topk values close {ok_v}, ids equal frac {same:.4f}, lse max err "
          f"{(l - lr).abs().max().item():.2e}")


def trace_call(fn, ctas=256):
    trace = torch.zeros(256 * 16 + 512, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    N.check(N.lib().nanospec_debug_set_trace(trace.data_ptr(), ctas), "trace")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    N.check(N.lib().nanospec_debug_set_trace(None, 0), "trace")
    t = trace[:256 * 16].view(256, 16).cpu().numpy().astype(np.int64)
    n = int((t[:, 0] > 0).sum())
    t = t[:n]
    t0 = t[:, 0].min()
    cyc, ns = t[:, 15] - t[:, 14], t[:, 6] - t[:, 0]
    ok = (t[:, 15] > 0) & (ns > 0)
    ghz = np.median(cyc[ok] / ns[ok]) if ok.any() else float("nan")
    print(f"  event {e0.elapsed_time(e1) * 1e3:.2f} us, {n} CTAs, SM clock {ghz:.3f} GHz")
    for e, name in enumerate(EV):
        c = t[:, e]
        c = c[c > 0]
        if len(c):
            r = (c - t0) / 1e3
            print(f"    {name:8s} n={len(c):3d} min {r.min():6.2f} med {np.median(r):6.2f} max {r.max():6.2f}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=60)
    ap.add_argument("--m", type=int, default=3072)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--mode", type=int, default=6)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    V, d = 128256, 4096
    N.check(N.lib().nanospec_debug_set_head_mode(args.mode), "mode")
    W = SI.bf16_weights(V, d, seed=0, device=dev)
    rng = np.random.default_rng(0)
    ids = rng.choice(V, args.m, replace=False).astype(np.int32)
    st = P.ActiveVocab(V, max(3072, args.m), device=dev)
    st.init(0, torch.as_tensor(ids, device=dev))
    H = SI.bf16_hidden(args.n, d, seed=1, device=dev).reshape(1, args.n, d)
    slots = st.read(0)["slots"]
    v, i, l, z = P.draft_logits_topk(st, W, H, args.k, debug_logits=True)
    torch.cuda.synchronize()
    print("head (pair mode)")
    ref_check(W, H[0], slots, v[0], i[0], l[0], z[0], args.k, "head")
    out = P.HeadOutputs(1, args.n, args.k, st.w_max, dev)
    for _ in range(3):
        P.draft_logits_topk(st, W, H, args.k, out=out)
    trace_call(lambda: P.draft_logits_topk(st, W, H, args.k, out=out))
    trace_call(lambda: P.draft_logits_topk(st, W, H, args.k, out=out))
    if os.environ.get("NANOSPEC_PAIR_DBG"):
        return
    # fused step vs update + head on a twin state
    pool = SI.disjoint_pools(V, 3072 + 126, 1, seed=5)[0]
    prompt, ups = SI.cyclic_fresh_updates(pool, 3072, 6)
    sa = P.ActiveVocab(V, 3072, device=dev)
    sb = P.ActiveVocab(V, 3072, device=dev)
    for s_ in (sa, sb):
        s_.init(0, torch.as_tensor(prompt, device=dev))
    print("fused step fused:", P.step_is_fused(sa, 60, 3, d, args.n, args.k))
    outa = P.HeadOutputs(1, args.n, args.k, 3072, dev)
    for j, (dr, vr) in enumerate(ups):
        dd, vv = torch.as_tensor(dr, device=dev), torch.as_tensor(vr, device=dev)
        va, ia, la = P.step(sa, 0, dd, vv, W, H[0], args.k, out=outa)
        sb.update(0, dd, vv)
        vb, ib, lb, _ = P.draft_logits_topk(sb, W, H, args.k)
        torch.cuda.synchronize()
        ra, rb = sa.read(0), sb.read(0)
        same_state = np.array_equal(ra["ids"], rb["ids"]) and np.array_equal(ra["bitmap"], rb["bitmap"])
        print(f"  step {j}: state equal {same_state}, topk ids equal {torch.equal(ia, ib)}, "
              f"values equal {torch.equal(va, vb)}, lse max diff {(la - lb).abs().max().item():.2e}")
        if j == 0:
            ref_check(W, H[0], rb["slots"], va[0], ia[0], la[0], None, args.k, "step")
    dd, vv = ups[0]
    trace_call(lambda: P.step(sa, 0, torch.as_tensor(dd, device=dev), torch.as_tensor(vv, device=dev), W, H[0],
                              args.k, out=outa))


if __name__ == "__main__":
    main()
