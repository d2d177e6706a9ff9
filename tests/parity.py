"""Comparison rules of the parity tests.

* state: ids, n_active, bitmap, ring and total bit-exact;
* logits: |z_gpu - z_ref| <= RTOL * max(|z_ref|, 2^-6 * A), A = sum |w h|
  (north_star: max relative error 2e-3 with bf16 inputs, fp32 accumulation);
* top-k ids exact at every rank, except where the two ids are a near-tie within
  2 * tol under the oracle's own logits; every GPU value must pass the logit
  tolerance for its own id;
* lse: |lse_gpu - lse_ref| <= RTOL * max(1, |lse_ref|).
"""
import numpy as np

RTOL = 2e-3
FLOOR = 2.0 ** -6


def tol(z_ref, A):
    return RTOL * np.maximum(np.abs(z_ref), FLOOR * A)


def check_logits(z_gpu, z_ref, A, what=""):
    z_gpu = np.asarray(z_gpu, np.float64)
    t = tol(z_ref, A)
    bad = np.abs(z_gpu - z_ref) > t
    assert not bad.any(), f"{what}: {bad.sum()} logits out of tolerance; worst " \
        f"{np.max(np.abs(z_gpu - z_ref) / np.maximum(t, 1e-300)):.3g}x tol"


def check_topk(v_gpu, id_gpu, z_ref, A, ids, v_ref, id_ref, what=""):
    """z_ref/A: [n, |I|] oracle logits over the active ids `ids` (ascending)."""
    v_gpu = np.asarray(v_gpu, np.float64)
    id_gpu = np.asarray(id_gpu)
    n, k = id_ref.shape
    pos = {int(g): j for j, g in enumerate(ids)}
    for i in range(n):
        for r in range(k):
            gr, gg = int(id_ref[i, r]), int(id_gpu[i, r])
            if gr == -1 or gg == -1:
                assert gr == gg, f"{what}: node {i} rank {r}: padding mismatch {gg} vs {gr}"
                assert np.isneginf(v_gpu[i, r])
                continue
            assert gg in pos, f"{what}: node {i} rank {r}: id {gg} not in the active set"
            jg, jr = pos[gg], pos[gr]
            t = tol(z_ref[i, jg], A[i, jg])
            assert abs(v_gpu[i, r] - z_ref[i, jg]) <= t, f"{what}: node {i} rank {r}: value off for id {gg}"
            if gg != gr:
                tie = 2 * max(t, tol(z_ref[i, jr], A[i, jr]))
                assert abs(z_ref[i, jg] - z_ref[i, jr]) <= tie, \
                    f"{what}: node {i} rank {r}: id {gg} vs oracle {gr} is not a near-tie"
        got = [int(x) for x in id_gpu[i] if x >= 0]
        assert len(set(got)) == len(got), f"{what}: node {i}: duplicate ids"


def check_lse(l_gpu, l_ref, what=""):
    l_gpu = np.asarray(l_gpu, np.float64)
    bad = np.abs(l_gpu - l_ref) > RTOL * np.maximum(1.0, np.abs(l_ref))
    assert not bad.any(), f"{what}: lse off at {np.nonzero(bad)[0][:5]}"
