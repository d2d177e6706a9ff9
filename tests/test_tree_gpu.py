"""The draft-tree bookkeeping (nanospec_tree_expand / nanospec_tree_rerank; Alg. 1
P:527-529) against the oracle's: (a) on the same random head
outputs, node by node; (b) a whole EAGLE-2-style round at the Llama-3.1-8B
shape -- one n = 1 head call and five n = 10 calls, each followed by an
expansion, then the rerank to 60 draft tokens -- every level checked against
the oracle's head + expansion of the same frontier, and the round then fed to
the fused decode step as C_draft."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from synthetic import inputs as SI

from parity import RTOL, check_lse, check_topk

pytestmark = pytest.mark.gpu


def _t(a, dt=torch.int32):
    return torch.as_tensor(np.asarray(a), dtype=dt, device="cuda").contiguous()


def test_expand_rerank_match_oracle(cuda_ok):
    from paper_2605_26444_b200 import DraftTree
    rng = np.random.default_rng(0)
    k, width, depth = 10, 10, 6
    tree = DraftTree(1 + k + (depth - 1) * width * k, width, "cuda")
    ref = O.OracleTree(tree.cap)
    n_front = 1
    for d in range(depth):
        val = -np.sort(-rng.normal(0, 2, (n_front, k)), axis=1).astype(np.float32)
        ids = rng.integers(0, 1000, (n_front, k)).astype(np.int32)
        lse = (val.max(axis=1) + rng.uniform(0.5, 3.0, n_front)).astype(np.float32)
        tree.expand(_t(val, torch.float32), _t(ids), _t(lse, torch.float32), width)
        fi, fs = ref.expand(val.astype(np.float64), ids, lse.astype(np.float64), width)
        torch.cuda.synchronize()
        assert np.array_equal(tree.front_index.cpu().numpy(), fi), f"level {d}: frontier"
        assert np.allclose(tree.front_score.cpu().numpy(), fs, rtol=1e-6, atol=1e-6), f"level {d}"
        n_front = width
    assert tree.n == ref.n
    assert np.array_equal(tree.id.cpu().numpy()[: tree.n], ref.id[: ref.n])
    assert np.array_equal(tree.parent.cpu().numpy()[: tree.n], ref.parent[: ref.n])
    assert np.allclose(tree.score.cpu().numpy()[: tree.n], ref.score[: ref.n], rtol=1e-6, atol=1e-6)
    idx, tok = tree.rerank(60)
    ridx, rtok = ref.rerank(60)
    assert np.array_equal(idx.cpu().numpy(), ridx) and np.array_equal(tok.cpu().numpy(), rtok)


def test_draft_round_llama_shape(cuda_ok):
    """A whole round on device at the Llama shape, checked level by level, then
    its 60 tree tokens + 3 verify tokens as one fused decode step."""
    from paper_2605_26444_b200 import ActiveVocab, DraftTree, HeadOutputs, draft_logits_topk, step
    V, d = SI.LLAMA["vocab"], SI.LLAMA["d_model"]
    W = SI.bf16_weights(V, d, seed=0, device="cuda")
    Wb = SI.bf16_bits(W)
    k, width, depth, m = 10, 10, 6, 60
    z = SI.Zipf(V)
    prompt, pre = SI.prompt_and_prefill(z, 4, 2000, 3)
    st = ActiveVocab(V, 3072)
    st.init(0, _t(prompt), _t(pre))
    ids = st.read(0)["ids"]
    tree = DraftTree(1 + k + (depth - 1) * width * k, width, "cuda")
    outs = {1: HeadOutputs(1, 1, k, 3072, "cuda"), width: HeadOutputs(1, width, k, 3072, "cuda")}
    Hs = [SI.bf16_hidden(1 if lvl == 0 else width, d, seed=200 + lvl, device="cuda") for lvl in range(depth)]
    for lvl in range(depth):
        nf = 1 if lvl == 0 else width
        front_before = None if lvl == 0 else (tree.front_index.cpu().numpy().copy(), tree.front_score.cpu().numpy().copy())
        v, i, l, _ = draft_logits_topk(st, W, Hs[lvl].reshape(1, nf, d), k, out=outs[nf])
        tree.expand(v[0], i[0], l[0], width)
        torch.cuda.synchronize()
        # the head of this level vs the oracle
        z_ref, A = O.logits(Wb, SI.bf16_bits(Hs[lvl]), ids)
        v_ref, id_ref = O.topk(z_ref, ids, k)
        lse_ref = O.lse(z_ref)
        check_topk(v[0].cpu().numpy(), i[0].cpu().numpy(), z_ref, A, ids, v_ref, id_ref, f"level {lvl}")
        check_lse(l[0].cpu().numpy(), lse_ref, f"level {lvl}")
        # the expansion of this frontier vs the oracle's, from the same frontier
        ref = O.OracleTree(tree.cap)
        ref.n = tree.n - nf * k  # the children land at the same pool indices
        fi, fs = ref.expand(v_ref, id_ref, lse_ref, width,
                            front_score=None if front_before is None else front_before[1].astype(np.float64),
                            front_index=None if front_before is None else front_before[0])
        got = tree.score.cpu().numpy()[tree.n - nf * k: tree.n]
        want = ref.score[tree.n - nf * k: tree.n]
        assert np.allclose(got, want, rtol=4 * RTOL, atol=4 * RTOL), f"level {lvl}: child scores"
        gf = tree.front_index.cpu().numpy()
        if not np.array_equal(gf, fi):  # only a near-tie may reorder the frontier
            gs = tree.front_score.cpu().numpy()
            assert np.allclose(np.sort(gs), np.sort(fs), rtol=4 * RTOL, atol=4 * RTOL), f"level {lvl}: frontier"
    idx, tok = tree.rerank(m)
    torch.cuda.synchronize()
    sc = tree.score.cpu().numpy()[: tree.n]
    order = np.lexsort((np.arange(tree.n), -sc))[:m]
    assert np.array_equal(idx.cpu().numpy(), order)
    # C_draft of the round (60 tree tokens) + 3 verify tokens -> the fused step, state vs the oracle
    ver = SI.decode_steps(z, 9, 1)[0][1]
    out = HeadOutputs(1, 60, k, 3072, "cuda")
    H = SI.bf16_hidden(60, d, seed=300, device="cuda")
    step(st, 0, tok, _t(ver), W, H, k, out=out)
    torch.cuda.synchronize()
    oref = O.OracleStream(V, 3072).init(prompt, pre).update(tok.cpu().numpy(), ver)
    assert np.array_equal(st.read(0)["ids"], oref.active()[0])
