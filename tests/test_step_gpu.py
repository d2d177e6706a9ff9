"""The fused decode step (nanospec_step: state update + head in one launch,
P:229-239 then P:527-528) against the oracle: after every step the state is
bit-exact (ids, n_active, bitmap, ring, total) and the top-k / lse of the
UPDATED active set pass the parity rules.  Covers the headline regime (|I| =
W_max, 63 ids enter and 63 leave per step), natural Zipf streams (I grows and
shrinks, duplicates inside the lists, ids already active), invalid ids, and
shapes that fall back to two launches."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from synthetic import inputs as SI

from parity import check_lse, check_topk

pytestmark = pytest.mark.gpu


def _t(a):
    return torch.as_tensor(np.asarray(a, np.int32), dtype=torch.int32, device="cuda").contiguous()


def _check_state(st, ref, what):
    got = st.read(0)
    ids, bm = ref.active()
    assert got["n_active"] == len(ids), what
    assert np.array_equal(got["ids"], ids), what
    assert np.array_equal(got["bitmap"], bm), what
    ring, total = ref.ring()
    assert got["total"] == total and np.array_equal(got["ring"], ring), what
    return ids


def _check_head(v, i, l, ids, Wb, H, k, what):
    z_ref, A = O.logits(Wb, SI.bf16_bits(H), ids)
    v_ref, id_ref = O.topk(z_ref, ids, k)
    check_topk(v[0].cpu().numpy(), i[0].cpu().numpy(), z_ref, A, ids, v_ref, id_ref, what)
    check_lse(l[0].cpu().numpy(), O.lse(z_ref), what)


@pytest.fixture(scope="module")
def llama():
    W = SI.bf16_weights(SI.LLAMA["vocab"], SI.LLAMA["d_model"], seed=0, device="cuda")
    return W, SI.bf16_bits(W)


def test_step_headline_regime(cuda_ok, llama):
    """|I| = W_max = 3072 every step: 63 fresh ids enter, 63 leave."""
    from paper_2605_26444_b200 import ActiveVocab, HeadOutputs, step
    W, Wb = llama
    V, d = W.shape
    Wm, n, k = 3072, 60, 10
    pool = SI.disjoint_pools(V, Wm + 126, 1, seed=5)[0]
    prompt, ups = SI.cyclic_fresh_updates(pool, Wm, 6)
    st = ActiveVocab(V, Wm)
    st.init(0, _t(prompt))
    ref = O.OracleStream(V, Wm).init(prompt)
    out = HeadOutputs(1, n, k, Wm, "cuda")
    for s, (dd, vv) in enumerate(ups):
        H = SI.bf16_hidden(n, d, seed=100 + s, device="cuda")
        v, i, l = step(st, 0, _t(dd), _t(vv), W, H, k, out=out)
        torch.cuda.synchronize()
        ref.update(dd, vv)
        ids = _check_state(st, ref, f"step {s}")
        assert len(ids) == Wm
        _check_head(v, i, l, ids, Wb, H, k, f"headline step {s}")


@pytest.mark.parametrize("n,k", [(60, 10), (10, 3), (1, 32)])
def test_step_natural_stream(cuda_ok, llama, n, k):
    """Zipf stream: repeated and already-active ids, I shrinking and growing."""
    from paper_2605_26444_b200 import ActiveVocab, HeadOutputs, step
    W, Wb = llama
    V, d = W.shape
    Wm = 3072
    z = SI.Zipf(V)
    prompt, pre = SI.prompt_and_prefill(z, 3, 600, 3)
    st = ActiveVocab(V, Wm)
    st.init(0, _t(prompt), _t(pre))
    ref = O.OracleStream(V, Wm).init(prompt, pre)
    out = HeadOutputs(1, n, k, Wm, "cuda")
    for s, (dd, vv) in enumerate(SI.decode_steps(z, 9, 60)):
        H = SI.bf16_hidden(n, d, seed=200 + s, device="cuda")
        v, i, l = step(st, 0, _t(dd), _t(vv), W, H, k, out=out)
        ref.update(dd, vv)
        if s % 6 == 5 or s < 2:
            torch.cuda.synchronize()
            ids = _check_state(st, ref, f"zipf step {s}")
            _check_head(v, i, l, ids, Wb, H, k, f"zipf n={n} k={k} step {s}")


def test_step_small_window_and_invalid_ids(cuda_ok, llama):
    """W_max = 256 (evictions every step), out-of-range ids (dropped, flagged)."""
    from paper_2605_26444_b200 import ActiveVocab, HeadOutputs, step
    W, Wb = llama
    V, d = W.shape
    Wm, n, k = 256, 16, 10
    rng = np.random.default_rng(4)
    st = ActiveVocab(V, Wm)
    prompt = rng.integers(0, V, 300)
    st.init(0, _t(prompt))
    ref = O.OracleStream(V, Wm).init(prompt)
    out = HeadOutputs(1, n, k, Wm, "cuda")
    for s in range(12):
        dd = rng.integers(0, V, 60)
        dd[::7] = dd[1]  # duplicates within the list
        if s == 5:
            dd[3] = V + 5  # invalid: dropped
        vv = rng.integers(0, V, 3)
        H = SI.bf16_hidden(n, d, seed=300 + s, device="cuda")
        v, i, l = step(st, 0, _t(dd), _t(vv), W, H, k, out=out)
        torch.cuda.synchronize()
        ref.update(dd, vv)
        ids = _check_state(st, ref, f"small-window step {s}")
        _check_head(v, i, l, ids, Wb, H, k, f"small-window step {s}")
    assert st.check() != 0  # the invalid id was flagged


def test_step_fallback_tiny(cuda_ok):
    """The tiny shape (d = 64: one K atom, so split-K 1) through nanospec_step:
    the oracle's state and top-k every step."""
    from paper_2605_26444_b200 import ActiveVocab, step
    V, d, Wm, n, k = 1000, 64, 256, 8, 10
    W = SI.bf16_weights(V, d, seed=0, device="cuda")
    Wb = SI.bf16_bits(W)
    z = SI.Zipf(V)
    prompt, pre = SI.prompt_and_prefill(z, 2, 200, 3)
    st = ActiveVocab(V, Wm)
    st.init(0, _t(prompt), _t(pre))
    ref = O.OracleStream(V, Wm).init(prompt, pre)
    for s, (dd, vv) in enumerate(SI.decode_steps(z, 5, 5, n_draft=8, k_ver=3)):
        H = SI.bf16_hidden(n, d, seed=1 + s, device="cuda")
        v, i, l = step(st, 0, _t(dd), _t(vv), W, H, k)
        torch.cuda.synchronize()
        ref.update(dd, vv)
        ids = _check_state(st, ref, f"tiny step {s}")
        _check_head(v, i, l, ids, Wb, H, k, f"tiny step {s}")


@pytest.mark.parametrize("mode", [-1, 0])
def test_step_launch_modes(cuda_ok, llama, mode):
    """The fused step with (-1) and without (0) programmatic dependent launch
    between its kernels: the oracle's state and top-k every step."""
    from paper_2605_26444_b200 import ActiveVocab, HeadOutputs, step, _native as N
    W, Wb = llama
    V, d = W.shape
    Wm, n, k = 3072, 60, 10
    cap = mode
    N.check(N.lib().nanospec_debug_set_head_mode(mode), "head mode")
    try:
        z = SI.Zipf(V)
        prompt, pre = SI.prompt_and_prefill(z, 8, 1500, 3)
        st = ActiveVocab(V, Wm)
        st.init(0, _t(prompt), _t(pre))
        ref = O.OracleStream(V, Wm).init(prompt, pre)
        out = HeadOutputs(1, n, k, Wm, "cuda")
        for s, (dd, vv) in enumerate(SI.decode_steps(z, 13, 4)):
            H = SI.bf16_hidden(n, d, seed=400 + s, device="cuda")
            v, i, l = step(st, 0, _t(dd), _t(vv), W, H, k, out=out)
            torch.cuda.synchronize()
            ref.update(dd, vv)
            ids = _check_state(st, ref, f"mode {cap} step {s}")
            _check_head(v, i, l, ids, Wb, H, k, f"mode {cap} step {s}")
    finally:
        N.check(N.lib().nanospec_debug_set_head_mode(-1), "head mode")


def test_step_many_back_to_back(cuda_ok, llama):
    """200 fused steps over 8 sequences captured in one CUDA graph (programmatic
    dependent launch between them), then every sequence checked."""
    from paper_2605_26444_b200 import ActiveVocab, HeadOutputs, step
    W, Wb = llama
    V, d = W.shape
    Wm, n, k, R, T = 3072, 60, 10, 8, 200
    pools = SI.disjoint_pools(V, Wm + 126, R, seed=9)
    sts, outs, refs, ups, Hs = [], [], [], [], SI.bf16_hidden(n, d, seed=7, device="cuda", batch=R)
    for r in range(R):
        prompt, u = SI.cyclic_fresh_updates(pools[r], Wm, T // R + 2)
        st = ActiveVocab(V, Wm)
        st.init(0, _t(prompt))
        sts.append(st)
        refs.append(O.OracleStream(V, Wm).init(prompt))
        outs.append(HeadOutputs(1, n, k, Wm, "cuda"))
        ups.append([(_t(a), _t(b), a, b) for a, b in u])
    stream = torch.cuda.Stream()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for s in range(T):
            r = s % R
            dd, vv, _, _ = ups[r][s // R]
            step(sts[r], 0, dd, vv, W, Hs[r], k, out=outs[r])
    g.replay()
    torch.cuda.synchronize()
    for r in range(R):
        for j in range(T // R):
            refs[r].update(ups[r][j][2], ups[r][j][3])
        ids = _check_state(sts[r], refs[r], f"seq {r}")
        v, i, l = outs[r].topk_logit, outs[r].topk_id, outs[r].lse
        _check_head(v, i, l, ids, Wb, Hs[r], k, f"graph seq {r}")


def test_step_host_buffers(cuda_ok, llama):
    """nanospec_step_host: packed host inputs -> step -> packed host results
    equals the oracle (the end-to-end call the bench times)."""
    from paper_2605_26444_b200 import ActiveVocab, StepHostIO, step_host
    W, Wb = llama
    V, d = W.shape
    Wm, n, k = 3072, 60, 10
    pool = SI.disjoint_pools(V, Wm + 126, 1, seed=21)[0]
    prompt, ups = SI.cyclic_fresh_updates(pool, Wm, 3)
    st = ActiveVocab(V, Wm)
    st.init(0, _t(prompt))
    ref = O.OracleStream(V, Wm).init(prompt)
    io = StepHostIO(n, d, 60, 3, k, Wm, "cuda")
    for s, (dd, vv) in enumerate(ups):
        H = SI.bf16_hidden(n, d, seed=500 + s, device="cuda")
        step_host(st, 0, io, io.pack_inputs(H, dd, vv), W, k)
        torch.cuda.synchronize()
        ref.update(dd, vv)
        ids = _check_state(st, ref, f"host step {s}")
        v, i, l = io.results()
        _check_head(v.unsqueeze(0), i.unsqueeze(0), l.unsqueeze(0), ids, Wb, H, k, f"host step {s}")


def test_step_host_pipelined(cuda_ok, llama):
    """nanospec_step_host_async (2 slots, input copies on a copy stream): four
    steps issued back to back without a sync, then every step's results (read
    from its slot once its event completed) and the final state equal the
    oracle's."""
    from paper_2605_26444_b200 import ActiveVocab, StepHostIO, step_host
    W, Wb = llama
    V, d = W.shape
    Wm, n, k = 3072, 60, 10
    pool = SI.disjoint_pools(V, Wm + 126, 1, seed=22)[0]
    prompt, ups = SI.cyclic_fresh_updates(pool, Wm, 4)
    st = ActiveVocab(V, Wm)
    st.init(0, _t(prompt))
    ref = O.OracleStream(V, Wm).init(prompt)
    io = StepHostIO(n, d, 60, 3, k, Wm, "cuda", slots=2)
    Hs = [SI.bf16_hidden(n, d, seed=700 + s, device="cuda") for s in range(len(ups))]
    blocks = [io.pack_inputs(Hs[s], dd, vv) for s, (dd, vv) in enumerate(ups)]
    torch.cuda.synchronize()
    got = []
    for s in range(len(ups)):
        step_host(st, 0, io, blocks[s], W, k)
        if s >= 1:  # the previous step's slot is reused two steps later: read it now
            io.ev_done[1 - io.slot].synchronize()
            got.append([x.clone() for x in io.results(1 - io.slot)])
    torch.cuda.synchronize()
    got.append([x.clone() for x in io.results()])
    for s, (dd, vv) in enumerate(ups):
        ref.update(dd, vv)
        ids = ref.active()[0]
        v, i, l = got[s]
        _check_head(v.unsqueeze(0), i.unsqueeze(0), l.unsqueeze(0), ids, Wb, Hs[s], k, f"pipelined step {s}")
    _check_state(st, ref, "pipelined host steps")


def test_step_qwen_shape(cuda_ok):
    """configs[2] shape (V = 152064, d = 3584): a 2k-token prompt with K_pre = 3,
    then fused steps on the natural active set."""
    from paper_2605_26444_b200 import ActiveVocab, HeadOutputs, step, step_is_fused
    W = SI.bf16_weights(SI.QWEN["vocab"], SI.QWEN["d_model"], seed=0, device="cuda")
    Wb = SI.bf16_bits(W)
    V, d = W.shape
    Wm, n, k = 3072, 60, 10
    z = SI.Zipf(V)
    prompt, pre = SI.prompt_and_prefill(z, 1, 2048, 3)
    st = ActiveVocab(V, Wm)
    st.init(0, _t(prompt), _t(pre))
    assert step_is_fused(st, 60, 3, d, n, k)
    ref = O.OracleStream(V, Wm).init(prompt, pre)
    out = HeadOutputs(1, n, k, Wm, "cuda")
    for s, (dd, vv) in enumerate(SI.decode_steps(z, 7, 6)):
        H = SI.bf16_hidden(n, d, seed=600 + s, device="cuda")
        v, i, l = step(st, 0, _t(dd), _t(vv), W, H, k, out=out)
        ref.update(dd, vv)
        if s in (0, 5):
            torch.cuda.synchronize()
            ids = _check_state(st, ref, f"qwen step {s}")
            _check_head(v, i, l, ids, Wb, H, k, f"qwen fused step {s}")


def test_step_other_sequence_of_a_batch(cuda_ok, llama):
    """nanospec_step on sequence 3 of a 5-sequence state: only that sequence's
    state changes; its top-k matches the oracle."""
    from paper_2605_26444_b200 import ActiveVocab, step
    W, Wb = llama
    V, d = W.shape
    Wm, n, k, B = 3072, 60, 10, 5
    z = SI.Zipf(V)
    st = ActiveVocab(V, Wm, batch=B)
    refs = []
    for b in range(B):
        p, pre = SI.prompt_and_prefill(z, 40 + b, 500 + 100 * b, 3)
        st.init(b, _t(p), _t(pre))
        refs.append(O.OracleStream(V, Wm).init(p, pre))
    before = [st.read(b)["ids"].copy() for b in range(B)]
    for s, (dd, vv) in enumerate(SI.decode_steps(z, 41, 3)):
        H = SI.bf16_hidden(n, d, seed=700 + s, device="cuda")
        v, i, l = step(st, 3, _t(dd), _t(vv), W, H, k)
        torch.cuda.synchronize()
        refs[3].update(dd, vv)
        got = st.read(3)
        ids, _ = refs[3].active()
        assert np.array_equal(got["ids"], ids), f"seq 3 step {s}"
        _check_head(v, i, l, ids, Wb, H, k, f"batch seq 3 step {s}")
    for b in (0, 1, 2, 4):
        assert np.array_equal(st.read(b)["ids"], before[b]), f"sequence {b} must be untouched"


@pytest.mark.parametrize("G", [2, 4])
def test_step_vocab_parallel_shards(cuda_ok, G):
    """The fused step on vocab shards (rank r owns ids g % G == r, rows W[r::G]),
    simulated on one GPU: every shard's state is bit-exact vs the oracle's shard
    and the merged per-shard top-k / lse equal the oracle's over the full set."""
    from paper_2605_26444_b200 import ActiveVocab, HeadOutputs, merge_topk, step, step_is_fused
    V, d, Wm, n, k = 40000, 1024, 3072, 60, 10
    W = SI.bf16_weights(V, d, seed=7, device="cuda")
    Wb = SI.bf16_bits(W)
    z = SI.Zipf(V)
    p, pre = SI.prompt_and_prefill(z, 4, 3000, 3)
    sts = []
    for r in range(G):
        st = ActiveVocab(V, Wm, shard_rank=r, n_shards=G)
        st.init(0, _t(p), _t(pre))
        sts.append(st)
    assert step_is_fused(sts[0], 60, 3, d, n, k)  # the sharded state takes the one-launch path
    ref = O.OracleStream(V, Wm).init(p, pre)
    Ws = [W[r::G].contiguous() for r in range(G)]
    outs = [HeadOutputs(1, n, k, Wm, "cuda") for _ in range(G)]
    for s, (dd, vv) in enumerate(SI.decode_steps(z, 5, 4)):
        H = SI.bf16_hidden(n, d, seed=800 + s, device="cuda")
        res = [step(sts[r], 0, _t(dd), _t(vv), Ws[r], H, k, out=outs[r]) for r in range(G)]
        ml, mi, mlse = merge_topk(torch.stack([x[0][0] for x in res]), torch.stack([x[1][0] for x in res]),
                                  torch.stack([x[2][0] for x in res]), k)
        torch.cuda.synchronize()
        ref.update(dd, vv)
        for r in range(G):
            ids_r, bm_r = ref.active(r, G)
            got = sts[r].read(0)
            assert np.array_equal(got["ids"], ids_r) and np.array_equal(got["bitmap"], bm_r), f"shard {r} step {s}"
        ids, _ = ref.active()
        z_ref, A = O.logits(Wb, SI.bf16_bits(H), ids)
        v_ref, id_ref = O.topk(z_ref, ids, k)
        check_topk(ml.cpu().numpy(), mi.cpu().numpy(), z_ref, A, ids, v_ref, id_ref, f"vp G={G} step {s}")
        check_lse(mlse.cpu().numpy(), O.lse(z_ref), f"vp G={G} step {s}")


def test_step_rule_r2_falls_back(cuda_ok, llama):
    """Rule R2 (unique-FIFO) has no fused path: nanospec_step runs update + head
    and still matches the oracle."""
    from paper_2605_26444_b200 import ActiveVocab, step, step_is_fused
    W, Wb = llama
    V, d = W.shape
    Wm, n, k = 1024, 16, 10
    z = SI.Zipf(V)
    p, pre = SI.prompt_and_prefill(z, 6, 800, 3)
    st = ActiveVocab(V, Wm, rule="unique_fifo")
    st.init(0, _t(p), _t(pre))
    assert not step_is_fused(st, 60, 3, d, n, k)
    ref = O.OracleStream(V, Wm, O.RULE_UNIQUE_FIFO).init(p, pre)
    for s, (dd, vv) in enumerate(SI.decode_steps(z, 8, 3)):
        H = SI.bf16_hidden(n, d, seed=900 + s, device="cuda")
        v, i, l = step(st, 0, _t(dd), _t(vv), W, H, k)
        torch.cuda.synchronize()
        ref.update(dd, vv)
        ids = _check_state(st, ref, f"R2 step {s}")
        _check_head(v, i, l, ids, Wb, H, k, f"R2 step {s}")
