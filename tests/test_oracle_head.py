"""Pins for the oracle's restricted LM head, top-k and lse (Eq. 2 restricted to
I; SelectDraftTokens).

The oracle is checked against library routines it does not use (numpy fp64 /
int64 matmul, numpy lexsort, scipy logsumexp, torch's bf16 conversion), exact
special cases (h = 0, one-hot h, integer-valued operands, duplicate rows,
single row) and the restriction property (pruned head == dense head masked to
I).  CPU only.
"""
import numpy as np
import pytest
import torch
from scipy.special import logsumexp

from oracle import oracle as O
from synthetic import inputs as SI


def _bits(t):
    return SI.bf16_bits(t)


def _f64(t):
    return t.to(torch.float64).numpy()


def test_bf16_decode_all_patterns():
    pats = torch.arange(0, 1 << 16, dtype=torch.int32).to(torch.int16).view(torch.bfloat16)
    ref = pats.to(torch.float64).numpy()
    bits = _bits(pats)
    for i in range(1 << 16):
        got = O.bf16_to_double(int(bits[i]))
        if np.isnan(ref[i]):
            assert np.isnan(got)
        else:
            assert got == ref[i]


def _case(V=200, d=48, n=5, seed=0):
    W = SI.bf16_weights(V, d, seed=seed)
    H = SI.bf16_hidden(n, d, seed=seed + 1)
    return W, H


def test_full_vocab_equals_dense_matmul():
    """I = [0, V) reduces to Eq. 2."""
    W, H = _case(V=300, d=64, n=7)
    ids = np.arange(300, dtype=np.int32)
    z, A = O.logits(_bits(W), _bits(H), ids)
    dense = _f64(H) @ _f64(W).T
    assert np.all(A >= np.abs(z) - 1e-15)
    np.testing.assert_allclose(z, dense, rtol=0, atol=1e-13 * max(1.0, A.max()))


def test_restriction_equals_masked_dense():
    """Pruned head == gathered rows of the dense head."""
    W, H = _case(V=257, d=40, n=3, seed=4)
    rng = np.random.default_rng(9)
    ids = np.sort(rng.choice(257, size=31, replace=False)).astype(np.int32)
    z, _ = O.logits(_bits(W), _bits(H), ids)
    dense = _f64(H) @ _f64(W).T
    np.testing.assert_allclose(z, dense[:, ids], rtol=0, atol=1e-13)


def test_ldw_padding_ignored():
    W, H = _case(V=50, d=32, n=2)
    Wp = torch.zeros(50, 40, dtype=torch.bfloat16)
    Wp[:, :32] = W
    Wp[:, 32:] = 7.0
    ids = np.arange(0, 50, 3, dtype=np.int32)
    z1, _ = O.logits(_bits(W), _bits(H), ids)
    z2, _ = O.logits(_bits(Wp), _bits(H), ids)
    assert np.array_equal(z1, z2)


def test_exact_special_cases():
    W, H = _case(V=64, d=32, n=4)
    ids = np.array([1, 5, 6, 40, 63], np.int32)
    # h = 0 -> z = 0 exactly
    z, _ = O.logits(_bits(W), _bits(torch.zeros(2, 32, dtype=torch.bfloat16)), ids)
    assert np.all(z == 0.0)
    # h = e_c -> z_j = W[I_j][c] exactly
    for c in (0, 7, 31):
        e = torch.zeros(1, 32, dtype=torch.bfloat16)
        e[0, c] = 1.0
        z, _ = O.logits(_bits(W), _bits(e), ids)
        assert np.array_equal(z[0], _f64(W)[ids, c])
    # single row I = {g} -> dot(W_g, h), against an integer-exact case
    Wi = SI.int_valued_bf16((64, 32), -16, 16, seed=3)
    Hi = SI.int_valued_bf16((4, 32), -16, 16, seed=4)
    z, _ = O.logits(_bits(Wi), _bits(Hi), ids)
    exact = Hi.to(torch.int64).numpy() @ Wi.to(torch.int64).numpy()[ids].T
    assert np.array_equal(z, exact.astype(np.float64))
    z1, _ = O.logits(_bits(Wi), _bits(Hi), np.array([40], np.int32))
    assert np.array_equal(z1[:, 0], exact[:, 3].astype(np.float64))


def _lexsort_topk(z, ids, k):
    n, m = z.shape
    vals = np.full((n, k), -np.inf)
    out = np.full((n, k), -1, np.int32)
    for i in range(n):
        order = np.lexsort((ids, -z[i]))  # primary: value desc, secondary: id asc
        t = min(k, m)
        vals[i, :t] = z[i, order[:t]]
        out[i, :t] = ids[order[:t]]
    return vals, out


@pytest.mark.parametrize("k", [1, 3, 10, 32])
def test_topk_matches_lexsort(k):
    W, H = _case(V=400, d=64, n=6, seed=k)
    rng = np.random.default_rng(k)
    ids = np.sort(rng.choice(400, size=57, replace=False)).astype(np.int32)
    z, _ = O.logits(_bits(W), _bits(H), ids)
    v, o = O.topk(z, ids, k)
    rv, ro = _lexsort_topk(z, ids, k)
    assert np.array_equal(o, ro) and np.array_equal(v, rv)


def test_topk_ties_and_padding():
    ids = np.array([3, 9, 12, 20], np.int32)
    z = np.zeros((2, 4))
    v, o = O.topk(z, ids, 6)  # h = 0: all tie -> ascending id, then padding
    assert o[0].tolist() == [3, 9, 12, 20, -1, -1]
    assert np.all(v[:, :4] == 0) and np.all(np.isneginf(v[:, 4:]))
    # duplicate rows -> equal logits -> the smaller id first (Q10)
    W = SI.bf16_weights(30, 16, seed=1)
    W[17] = W[4]
    H = SI.bf16_hidden(3, 16, seed=2)
    ids = np.array([4, 10, 17, 25], np.int32)
    z, _ = O.logits(_bits(W), _bits(H), ids)
    assert np.array_equal(z[:, 0], z[:, 2])
    v, o = O.topk(z, ids, 4)
    for i in range(3):
        lst = o[i].tolist()
        assert lst.index(4) < lst.index(17)


def test_lse_pins():
    W, H = _case(V=120, d=32, n=5, seed=6)
    ids = np.arange(0, 120, 2, dtype=np.int32)
    z, _ = O.logits(_bits(W), _bits(H), ids)
    l = O.lse(z)
    np.testing.assert_allclose(l, logsumexp(z, axis=1), rtol=0, atol=1e-12)
    np.testing.assert_allclose(np.exp(z - l[:, None]).sum(1), 1.0, rtol=0, atol=1e-12)
    z0 = np.zeros((2, 60))
    np.testing.assert_allclose(O.lse(z0), np.log(60.0), rtol=0, atol=1e-14)
