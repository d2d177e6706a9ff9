"""Round-2 parity cases at the full sizes BASELINE.json names, in the launch
configurations the bench times, against the oracle (tests/parity.py rules):

* dp64-shaped: a batch of sequences whose row tiles outnumber the SMs (the
  persistent split-K = 1 path of the head), Zipf and exact-3072 active sets;
* vp32k-shaped: a 32k-slot window over a 32k-token Zipf stream (~11k active
  ids, 256 row-tile capacity);
* the FR-Spec-style static 32k id set through nanospec_logits_topk_ids;
* the fused decode step's logits, element by element (nanospec_step_debug);
* one scratch reused across calls with different k / n;
* the fused step while another stream keeps the SMs busy (no launch of the
  head path waits for a CTA that may not be resident).
Every call goes through the C ABI."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from synthetic import inputs as SI

from parity import check_logits, check_lse, check_topk

pytestmark = pytest.mark.gpu


def _t(a):
    return torch.as_tensor(np.asarray(a, np.int32), dtype=torch.int32, device="cuda").contiguous()


@pytest.fixture(scope="module")
def llama():
    W = SI.bf16_weights(SI.LLAMA["vocab"], SI.LLAMA["d_model"], seed=0, device="cuda")
    return W, SI.bf16_bits(W)


def _check(v, i, l, ids, Wb, H, k, what, z=None):
    z_ref, A = O.logits(Wb, SI.bf16_bits(H), ids)
    if z is not None:
        check_logits(z, z_ref, A, what)
    v_ref, id_ref = O.topk(z_ref, ids, k)
    check_topk(v, i, z_ref, A, ids, v_ref, id_ref, what)
    check_lse(l, O.lse(z_ref), what)


def test_dp64_shaped_batch(cuda_ok, llama):
    """BASELINE configs[3] shape on one GPU: 16 Llama-shape sequences at W_max
    3072 (16 x 24 = 384 row tiles > 148 SMs: split-K 1, persistent CTAs), half
    of them at exactly |I| = 3072, half on natural Zipf streams; every
    sequence's top-k / lse and sequence 0's logits vs the oracle."""
    from paper_2605_26444_b200 import ActiveVocab, draft_logits_topk
    W, Wb = llama
    V, d = W.shape
    B, n, k, Wm = 16, 60, 10, 3072
    st = ActiveVocab(V, Wm, batch=B)
    z = SI.Zipf(V)
    pools = SI.disjoint_pools(V, Wm + 126, B // 2, seed=21)
    for b in range(B):
        if b % 2 == 0:
            prompt, _ = SI.cyclic_fresh_updates(pools[b // 2], Wm, 1)
            st.init(b, _t(prompt))
        else:
            p, pre = SI.prompt_and_prefill(z, 40 + b, 1000 + 60 * b, 3)
            st.init(b, _t(p), _t(pre))
    H = SI.bf16_hidden(n, d, seed=23, device="cuda", batch=B)
    v, i, l, zz = draft_logits_topk(st, W, H, k, debug_logits=True)
    torch.cuda.synchronize()
    for b in range(B):
        got = st.read(b)
        ids = got["slots"]
        assert got["n_active"] == (Wm if b % 2 == 0 else got["n_active"])
        zb = zz[b, :, : len(ids)].cpu().numpy() if b in (0, 1) else None
        _check(v[b].cpu().numpy(), i[b].cpu().numpy(), l[b].cpu().numpy(), ids, Wb, H[b], k, f"dp seq {b}", zb)


def test_vp32k_shaped_window(cuda_ok, llama):
    """BASELINE configs[4] active set on one GPU: W_max = 32768 over a
    32768-token Zipf stream (~11.4k active ids), then decode updates."""
    from paper_2605_26444_b200 import ActiveVocab, draft_logits_topk
    W, Wb = llama
    V, d = W.shape
    Wm, n, k = 32768, 60, 10
    zf = SI.Zipf(V)
    prompt, _ = SI.prompt_and_prefill(zf, 1, Wm, 0)
    st = ActiveVocab(V, Wm)
    st.init(0, _t(prompt))
    ref = O.OracleStream(V, Wm).init(prompt)
    for dd, vv in SI.decode_steps(zf, 7, 3):
        st.update(0, _t(dd), _t(vv))
        ref.update(dd, vv)
    got = st.read(0)
    ids_ref, _ = ref.active()
    assert np.array_equal(got["ids"], ids_ref)
    assert 9000 < got["n_active"] < 14000  # the ~11k regime of SURVEY 8(d)
    H = SI.bf16_hidden(n, d, seed=31, device="cuda")
    v, i, l, zz = draft_logits_topk(st, W, H.reshape(1, n, d), k, debug_logits=True)
    torch.cuda.synchronize()
    ids = got["slots"]
    _check(v[0].cpu().numpy(), i[0].cpu().numpy(), l[0].cpu().numpy(), ids, Wb, H, k, "vp32k window",
           zz[0, :, : len(ids)].cpu().numpy())


def test_static_32k_set(cuda_ok, llama):
    """FR-Spec-style fixed 32768-id set through the explicit-list
    entry point: 256 row tiles, logits element by element."""
    from paper_2605_26444_b200 import logits_topk_ids
    W, Wb = llama
    V, d = W.shape
    ids = np.sort(np.random.default_rng(11).permutation(V)[:32768]).astype(np.int32)
    n, k = 16, 10
    H = SI.bf16_hidden(n, d, seed=41, device="cuda")
    v, i, l, zz = logits_topk_ids(_t(ids), _t([len(ids)]), W, H, k, debug_logits=True)
    torch.cuda.synchronize()
    _check(v[0].cpu().numpy(), i[0].cpu().numpy(), l[0].cpu().numpy(), ids, Wb, H, k, "static 32k set",
           zz[0, :, : len(ids)].cpu().numpy())


@pytest.mark.parametrize("regime", ["headline", "zipf"])
def test_fused_step_logits_elementwise(cuda_ok, llama, regime):
    """nanospec_step_debug: every row the fused launch streamed -- the
    pre-update slots and the update-list entries -- has the oracle's logit; the
    rows that count are exactly I after the update; top-k / lse of that set."""
    from paper_2605_26444_b200 import ActiveVocab, HeadOutputs, step_debug
    W, Wb = llama
    V, d = W.shape
    Wm, n, k = 3072, 60, 10
    st = ActiveVocab(V, Wm)
    if regime == "headline":
        pool = SI.disjoint_pools(V, Wm + 126, 1, seed=5)[0]
        prompt, ups = SI.cyclic_fresh_updates(pool, Wm, 3)
        st.init(0, _t(prompt))
        ref = O.OracleStream(V, Wm).init(prompt)
    else:
        zf = SI.Zipf(V)
        prompt, pre = SI.prompt_and_prefill(zf, 3, 1500, 3)
        ups = SI.decode_steps(zf, 9, 3)
        st.init(0, _t(prompt), _t(pre))
        ref = O.OracleStream(V, Wm).init(prompt, pre)
    out = HeadOutputs(1, n, k, Wm, "cuda")
    for s, (dd, vv) in enumerate(ups):
        slots_before = st.read(0)["slots"]
        H = SI.bf16_hidden(n, d, seed=50 + s, device="cuda")
        v, i, l, dbg = step_debug(st, 0, _t(dd), _t(vv), W, H, k, out=out)
        torch.cuda.synchronize()
        ref.update(dd, vv)
        ids_new, _ = ref.active()
        assert np.array_equal(st.read(0)["ids"], ids_new), f"{regime} step {s}: state"
        dbg = dbg.cpu().numpy()
        entries = np.concatenate([np.asarray(dd, np.int32), np.asarray(vv, np.int32)])
        rows = np.concatenate([slots_before, entries])
        cols = np.concatenate([np.arange(len(slots_before)), Wm + np.arange(len(entries))])
        valid = (rows >= 0) & (rows < V)
        z_ref, A = O.logits(Wb, SI.bf16_bits(H), rows[valid])
        check_logits(dbg[:, cols[valid]], z_ref, A, f"{regime} step {s}: streamed rows")
        _check(v[0].cpu().numpy(), i[0].cpu().numpy(), l[0].cpu().numpy(), ids_new, Wb, H, k, f"{regime} step {s}")


def test_scratch_reuse_across_k_and_n(cuda_ok, llama):
    """One head scratch shared by calls with different k and n (k = 32 / n = 1,
    then k = 10 / n = 60, then k = 32 again): every call matches the oracle."""
    from paper_2605_26444_b200 import ActiveVocab, HeadOutputs, draft_logits_topk
    W, Wb = llama
    V, d = W.shape
    ids = np.random.default_rng(3).choice(V, 3072, replace=False)
    st = ActiveVocab(V, 3072)
    st.init(0, _t(ids))
    slots = st.read(0)["slots"]
    shared = HeadOutputs(1, 60, 32, 3072, "cuda").scratch
    for n, k in ((1, 32), (60, 10), (60, 32), (10, 1)):
        out = HeadOutputs(1, n, k, 3072, "cuda")
        out.scratch = shared
        H = SI.bf16_hidden(n, d, seed=60 + n + k, device="cuda")
        v, i, l, _ = draft_logits_topk(st, W, H.reshape(1, n, d), k, out=out)
        torch.cuda.synchronize()
        _check(v[0].cpu().numpy(), i[0].cpu().numpy(), l[0].cpu().numpy(), slots, Wb, H, k, f"reuse n={n} k={k}")


def test_step_with_busy_sms(cuda_ok, llama):
    """The paper runs its gather on a second stream beside the backbone
    (P:251-256): here a long GEMM loop occupies SMs on another stream while the
    fused step runs; it completes and matches the oracle."""
    from paper_2605_26444_b200 import ActiveVocab, HeadOutputs, step
    W, Wb = llama
    V, d = W.shape
    Wm, n, k = 3072, 60, 10
    pool = SI.disjoint_pools(V, Wm + 126, 1, seed=8)[0]
    prompt, ups = SI.cyclic_fresh_updates(pool, Wm, 3)
    st = ActiveVocab(V, Wm)
    st.init(0, _t(prompt))
    ref = O.OracleStream(V, Wm).init(prompt)
    out = HeadOutputs(1, n, k, Wm, "cuda")
    a = torch.randn(4096, 4096, dtype=torch.bfloat16, device="cuda")
    torch.cuda.synchronize()
    busy, mine = torch.cuda.Stream(), torch.cuda.Stream()
    for s, (dd, vv) in enumerate(ups):
        H = SI.bf16_hidden(n, d, seed=70 + s, device="cuda")
        with torch.cuda.stream(busy):
            for _ in range(40):
                a = (a @ a).clamp_(-1, 1)
        with torch.cuda.stream(mine):
            v, i, l = step(st, 0, _t(dd), _t(vv), W, H, k, out=out)
        torch.cuda.synchronize()
        ref.update(dd, vv)
        ids_new, _ = ref.active()
        assert np.array_equal(st.read(0)["ids"], ids_new)
        _check(v[0].cpu().numpy(), i[0].cpu().numpy(), l[0].cpu().numpy(), ids_new, Wb, H, k, f"busy step {s}")


def test_repack_variant_matches(cuda_ok, llama):
    """The paper's repack design as built: after every update the
    changed slots are re-copied (nanospec_repack) and the head over the packed
    rows gives bit-identical results to the fused direct gather; the packed
    rows equal W_head[ids]."""
    from paper_2605_26444_b200 import ActiveVocab, HeadOutputs, PackedHead, draft_logits_topk
    W, Wb = llama
    V, d = W.shape
    Wm, n, k = 3072, 60, 10
    zf = SI.Zipf(V)
    prompt, pre = SI.prompt_and_prefill(zf, 6, 1800, 3)
    st = ActiveVocab(V, Wm)
    st.init(0, _t(prompt), _t(pre))
    ph = PackedHead(st, d, "cuda")
    o1, o2 = HeadOutputs(1, n, k, Wm, "cuda"), HeadOutputs(1, n, k, Wm, "cuda")
    copy = torch.cuda.Stream()
    for s, (dd, vv) in enumerate(SI.decode_steps(zf, 12, 4)):
        st.update(0, _t(dd), _t(vv))
        ev = torch.cuda.Event()
        ev.record()
        with torch.cuda.stream(copy):  # the paper's copy stream
            copy.wait_event(ev)
            ph.refresh(0, W)
        torch.cuda.current_stream().wait_stream(copy)
        H = SI.bf16_hidden(n, d, seed=90 + s, device="cuda").reshape(1, n, d)
        v1, i1, l1, _ = draft_logits_topk(st, W, H, k, out=o1)
        v2, i2, l2 = ph.head(H, k, o2)
        torch.cuda.synchronize()
        assert torch.equal(i1, i2) and torch.equal(v1, v2) and torch.equal(l1, l2), f"step {s}"
        slots = st.read(0)["slots"]
        assert torch.equal(ph.packed[0, : len(slots)], W[torch.as_tensor(slots, device="cuda").long()])


def test_persistent_odd_tile_count(cuda_ok, llama):
    """The persistent split-K-1 mode with 256-row units when a sequence has an
    odd number of row tiles (W_max 2900 -> 23 tiles, 8 sequences: 184 tiles >
    148 SMs): the last unit of every sequence holds one tile."""
    from paper_2605_26444_b200 import ActiveVocab, draft_logits_topk
    W, Wb = llama
    V, d = W.shape
    B, n, k, Wm = 8, 60, 10, 2900
    st = ActiveVocab(V, Wm, batch=B)
    rng = np.random.default_rng(17)
    for b in range(B):
        st.init(b, _t(rng.choice(V, Wm - 37 * b, replace=False)))
    H = SI.bf16_hidden(n, d, seed=29, device="cuda", batch=B)
    v, i, l, zz = draft_logits_topk(st, W, H, k, debug_logits=True)
    torch.cuda.synchronize()
    for b in (0, 3, 7):
        ids = st.read(b)["slots"]
        _check(v[b].cpu().numpy(), i[b].cpu().numpy(), l[b].cpu().numpy(), ids, Wb, H[b], k, f"odd tiles seq {b}",
               zz[b, :, : len(ids)].cpu().numpy())
