"""Head (a3+a4+a5) vs the oracle: logits (debug output), top-k ids/values and
lse under the tolerances of tests/parity.py, for both contraction kernels, at
the tiny, Llama-3.1-8B and Qwen-2.5-7B shapes, ragged active-set sizes and the
exact special cases (integer-valued operands, one-hot h, h = 0, duplicate
rows).  Every call goes through the C ABI."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from synthetic import inputs as SI

from parity import check_logits, check_lse, check_topk

pytestmark = pytest.mark.gpu

IMPLS = ["simt", "tc"]


def _t(a):
    return torch.as_tensor(np.asarray(a, np.int32), dtype=torch.int32, device="cuda").contiguous()


def _state_with_ids(V, ids, w_max=None):
    from paper_2605_26444_b200 import ActiveVocab
    ids = np.asarray(ids, np.int32)
    st = ActiveVocab(V, w_max or max(len(ids), 1))
    st.init(0, _t(ids))
    return st


def _run(st, W, H, k, impl):
    from paper_2605_26444_b200 import draft_logits_topk
    from paper_2605_26444_b200._native import NanoSpecError, EUNSUPPORTED
    try:
        v, i, l, z = draft_logits_topk(st, W, H.reshape(1, -1, W.shape[1]), k, debug_logits=True, impl=impl)
    except NanoSpecError as e:
        if e.status == EUNSUPPORTED and impl == "tc":
            pytest.skip("tensor-core head not built for this shape")
        raise
    torch.cuda.synchronize()
    return v[0].cpu().numpy(), i[0].cpu().numpy(), l[0].cpu().numpy(), z[0].cpu().numpy()


def _full_check(st, W, Wbits, H, k, impl, what, exact=False):
    got = st.read(0)
    ids = got["slots"]  # device row order of the debug logits
    assert np.array_equal(np.sort(ids), got["ids"])
    z_ref, A = O.logits(Wbits, SI.bf16_bits(H), ids)
    v, i, l, z = _run(st, W, H, k, impl)
    m = len(ids)
    if exact:
        assert np.array_equal(z[:, :m].astype(np.float64), z_ref), what
    else:
        check_logits(z[:, :m], z_ref, A, what)
    v_ref, id_ref = O.topk(z_ref, ids, k)
    if exact:
        assert np.array_equal(i, id_ref), what
    check_topk(v, i, z_ref, A, ids, v_ref, id_ref, what)
    check_lse(l, O.lse(z_ref), what)
    return z_ref, ids, v, i, l


@pytest.fixture(scope="module")
def llama():
    W = SI.bf16_weights(SI.LLAMA["vocab"], SI.LLAMA["d_model"], seed=0, device="cuda")
    return W, SI.bf16_bits(W)


@pytest.fixture(scope="module")
def qwen():
    W = SI.bf16_weights(SI.QWEN["vocab"], SI.QWEN["d_model"], seed=0, device="cuda")
    return W, SI.bf16_bits(W)


@pytest.mark.parametrize("impl", IMPLS)
def test_tiny_config(cuda_ok, impl):
    from paper_2605_26444_b200 import ActiveVocab
    V, d = 1000, 64
    W = SI.bf16_weights(V, d, seed=0, device="cuda")
    Wb = SI.bf16_bits(W)
    z = SI.Zipf(V)
    prompt, pre = SI.prompt_and_prefill(z, 2, 200, 3)
    for w_max in (3072, 64):
        st = ActiveVocab(V, w_max)
        st.init(0, _t(prompt), _t(pre))
        for step, (dd, vv) in enumerate(SI.decode_steps(z, 5, 5, n_draft=8, k_ver=3)):
            st.update(0, _t(dd), _t(vv))
            H = SI.bf16_hidden(8, d, seed=1 + step, device="cuda")
            _full_check(st, W, Wb, H, 10, impl, f"tiny W={w_max} step {step}")


@pytest.mark.parametrize("impl", IMPLS)
@pytest.mark.parametrize("n,k,m", [(60, 10, 3072), (1, 32, 3072), (10, 1, 1665), (60, 10, 129), (8, 10, 1),
                                   (60, 32, 3071), (16, 5, 200), (33, 7, 2500)])
def test_llama_shape(cuda_ok, llama, impl, n, k, m):
    W, Wb = llama
    rng = np.random.default_rng(n * 1000 + m)
    ids = np.sort(rng.choice(W.shape[0], size=m, replace=False))
    st = _state_with_ids(W.shape[0], rng.permutation(ids), w_max=3072)
    H = SI.bf16_hidden(n, W.shape[1], seed=n + m, device="cuda")
    _full_check(st, W, Wb, H, k, impl, f"llama n={n} k={k} |I|={m}")


@pytest.mark.parametrize("impl", IMPLS)
def test_qwen_natural_active_set(cuda_ok, qwen, impl):
    """configs[2]: 2k-token Zipf prompt + K_pre = 3, then decode updates; the head
    runs on the natural (ragged, ~2-3k) active set."""
    from paper_2605_26444_b200 import ActiveVocab
    W, Wb = qwen
    V = W.shape[0]
    z = SI.Zipf(V)
    prompt, pre = SI.prompt_and_prefill(z, 1, 2048, 3)
    st = ActiveVocab(V, 3072)
    st.init(0, _t(prompt), _t(pre))
    for s, (dd, vv) in enumerate(SI.decode_steps(z, 7, 40)):
        st.update(0, _t(dd), _t(vv))
        if s in (0, 39):
            H = SI.bf16_hidden(60, W.shape[1], seed=s, device="cuda")
            _full_check(st, W, Wb, H, 10, impl, f"qwen step {s}")


@pytest.mark.parametrize("impl", IMPLS)
def test_exact_integer_valued(cuda_ok, impl):
    """|w|,|h| <= 16 integers, d = 4096: every fp32 partial sum is an integer
    below 2^24, so any summation order is exact -> bit-exact logits and ids."""
    V, d = 20000, 4096
    W = SI.int_valued_bf16((V, d), -16, 16, seed=3, device="cuda")
    Wb = SI.bf16_bits(W)
    rng = np.random.default_rng(0)
    ids = rng.choice(V, size=2000, replace=False)
    st = _state_with_ids(V, ids, w_max=2048)
    H = SI.int_valued_bf16((60, d), -16, 16, seed=4, device="cuda")
    _full_check(st, W, Wb, H, 32, impl, "integer-valued", exact=True)


@pytest.mark.parametrize("impl", IMPLS)
def test_exact_one_hot_zero_and_duplicates(cuda_ok, impl):
    V, d = 4000, 512
    W = SI.bf16_weights(V, d, seed=5, device="cuda")
    W[1234] = W[77]  # duplicate rows -> bit-equal logits -> ascending id first (Q10)
    W[3999] = W[77]
    Wb = SI.bf16_bits(W)
    ids = np.array(sorted(set(np.random.default_rng(1).choice(V, 700, replace=False).tolist()) | {77, 1234, 3999}))
    st = _state_with_ids(V, ids, w_max=1024)
    H = torch.zeros(4, d, dtype=torch.bfloat16, device="cuda")
    for i, c in enumerate((0, 5, 300)):
        H[i + 1, c] = 1.0  # one-hot rows: z_j = W[I_j][c] exactly
    z_ref, ids_o, v, i, l = _full_check(st, W, Wb, H, 32, impl, "one-hot/zero", exact=True)
    assert i[0].tolist() == sorted(ids_o.tolist())[:32]  # h = 0: all tie -> smallest ids (whatever the slot order)
    assert abs(l[0] - np.log(len(ids_o))) < 1e-5
    Hr = SI.bf16_hidden(6, d, seed=9, device="cuda")
    _, _, _, zz = _run(st, W, Hr, 32, impl)
    pos = {int(g): j for j, g in enumerate(ids_o)}
    assert np.array_equal(zz[:, pos[77]], zz[:, pos[1234]]) and np.array_equal(zz[:, pos[77]], zz[:, pos[3999]])
    v2, i2, _, _ = _run(st, W, Hr, 32, impl)
    for r in range(6):
        lst = i2[r].tolist()
        if 77 in lst and 1234 in lst:
            assert lst.index(77) < lst.index(1234)


@pytest.mark.parametrize("impl", IMPLS)
def test_batch_of_sequences(cuda_ok, llama, impl):
    """dp config: one head call over B independent sequences with different
    active sets."""
    from paper_2605_26444_b200 import ActiveVocab, draft_logits_topk
    W, Wb = llama
    V, d = W.shape
    B, n, k = 5, 60, 10
    z = SI.Zipf(V)
    st = ActiveVocab(V, 3072, batch=B)
    for b in range(B):
        p, pre = SI.prompt_and_prefill(z, 30 + b, 300 * (b + 1), 3)
        st.init(b, _t(p), _t(pre))
    H = SI.bf16_hidden(n, d, seed=3, device="cuda", batch=B)
    v, i, l, _ = draft_logits_topk(st, W, H, k, impl=impl)
    torch.cuda.synchronize()
    for b in range(B):
        ids = st.read(b)["slots"]
        z_ref, A = O.logits(Wb, SI.bf16_bits(H[b]), ids)
        v_ref, id_ref = O.topk(z_ref, ids, k)
        check_topk(v[b].cpu().numpy(), i[b].cpu().numpy(), z_ref, A, ids, v_ref, id_ref, f"seq {b}")
        check_lse(l[b].cpu().numpy(), O.lse(z_ref), f"seq {b}")


@pytest.fixture
def head_mode():
    """Launch the head's kernels with (-1) or without (0) programmatic dependent
    launch for one test (debug ABI), then back to the default."""
    from paper_2605_26444_b200 import _native as N

    def set_mode(m):
        N.check(N.lib().nanospec_debug_set_head_mode(m), "nanospec_debug_set_head_mode")

    yield set_mode
    set_mode(-1)


@pytest.mark.parametrize("mode", [-1, 0])
@pytest.mark.parametrize("n,k,m", [(60, 10, 3072), (1, 32, 3072), (60, 10, 129), (33, 7, 2500), (4, 10, 1),
                                   (100, 10, 3072), (200, 3, 1000)])
def test_tc_reduction_modes(cuda_ok, llama, head_mode, mode, n, k, m):
    """The two-kernel tensor-core head (K-split partials, then the select
    kernel) with and without programmatic dependent launch, node counts up to
    UMMA N = 256, against the oracle."""
    W, Wb = llama
    head_mode(mode)
    rng = np.random.default_rng(7 * n + m)
    ids = rng.choice(W.shape[0], size=m, replace=False)
    st = _state_with_ids(W.shape[0], ids, w_max=3072)
    H = SI.bf16_hidden(n, W.shape[1], seed=n + m + 1, device="cuda")
    _full_check(st, W, Wb, H, k, "tc", f"mode {mode} n={n} k={k} |I|={m}")
    # repeated calls reuse the scratch
    _full_check(st, W, Wb, H, k, "tc", f"mode {mode} repeat")


@pytest.mark.parametrize("mode", [-1, 0])
def test_tc_modes_bit_exact(cuda_ok, head_mode, mode):
    """Integer-valued operands: bit-exact logits and ids (the K-split partials
    are integers, summed in any order exactly)."""
    head_mode(mode)
    V, d = 20000, 4096
    W = SI.int_valued_bf16((V, d), -16, 16, seed=3, device="cuda")
    Wb = SI.bf16_bits(W)
    ids = np.random.default_rng(2).choice(V, size=3000, replace=False)
    st = _state_with_ids(V, ids, w_max=3072)
    H = SI.int_valued_bf16((60, d), -16, 16, seed=4, device="cuda")
    _full_check(st, W, Wb, H, 10, "tc", f"integer-valued mode {mode}", exact=True)


def test_large_active_set(cuda_ok, llama):
    """A 16k window with 11000 active ids (the vp32k regime on one GPU): 128 row
    tiles, 86 of them live: split-K 1 and several select rounds."""
    W, Wb = llama
    rng = np.random.default_rng(11)
    ids = rng.choice(W.shape[0], size=11000, replace=False)
    st = _state_with_ids(W.shape[0], ids, w_max=16384)
    H = SI.bf16_hidden(60, W.shape[1], seed=12, device="cuda")
    _full_check(st, W, Wb, H, 10, "tc", "|I|=11000")
