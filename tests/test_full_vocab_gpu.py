"""Full-vocabulary special case (I = [0, V) reduces to Eq. 2) and the
vocab-parallel merge.

* our head over ids = [0, V) vs cuBLAS (torch.matmul, fp32 out) + torch.topk --
  a dense reference independent of our kernels -- and vs the oracle on sampled
  nodes;
* G shards simulated on one GPU (cyclic g % G == rank, weights W[rank::G]),
  then nanospec_merge_topk: equal to the unsharded result bit-exactly."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from synthetic import inputs as SI

from parity import check_logits, check_lse, check_topk

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("impl", ["simt", "tc"])
def test_dense_full_vocab_llama(cuda_ok, impl):
    from paper_2605_26444_b200 import logits_topk_ids
    from paper_2605_26444_b200._native import NanoSpecError, EUNSUPPORTED
    V, d = SI.LLAMA["vocab"], SI.LLAMA["d_model"]
    W = SI.bf16_weights(V, d, seed=0, device="cuda")
    n, k = 4, 10
    H = SI.bf16_hidden(n, d, seed=2, device="cuda")
    ids = torch.arange(V, dtype=torch.int32, device="cuda")
    nid = torch.tensor([V], dtype=torch.int32, device="cuda")
    try:
        v, i, l, z = logits_topk_ids(ids, nid, W, H, k, debug_logits=True, impl=impl)
    except NanoSpecError as e:
        if e.status == EUNSUPPORTED:
            pytest.skip("tensor-core head not built for this shape")
        raise
    dense = torch.matmul(H.float(), W.float().t())  # cuBLAS fp32 (bf16 values exact in fp32)
    tv, ti = torch.topk(dense, k, dim=1)
    torch.cuda.synchronize()
    zr = dense.cpu().numpy().astype(np.float64)
    A = torch.matmul(H.float().abs(), W.float().abs().t()).cpu().numpy().astype(np.float64)
    check_logits(z[0].cpu().numpy(), zr, A, "dense vs cuBLAS")
    # top-k vs cuBLAS+topk (ties within tolerance allowed), then vs the oracle on 2 nodes
    ids_np = np.arange(V, dtype=np.int32)
    check_topk(v[0].cpu().numpy(), i[0].cpu().numpy(), zr, A, ids_np, tv.cpu().numpy().astype(np.float64),
               ti.cpu().numpy().astype(np.int32), "dense vs torch.topk")
    Hb = SI.bf16_bits(H[:2])
    z_ref, A_ref = O.logits(SI.bf16_bits(W), Hb, ids_np)
    v_ref, id_ref = O.topk(z_ref, ids_np, k)
    check_topk(v[0, :2].cpu().numpy(), i[0, :2].cpu().numpy(), z_ref, A_ref, ids_np, v_ref, id_ref, "dense vs oracle")
    check_lse(l[0, :2].cpu().numpy(), O.lse(z_ref), "dense lse")


@pytest.mark.parametrize("impl", ["simt", "tc"])
@pytest.mark.parametrize("G", [2, 8])
def test_vocab_parallel_merge(cuda_ok, impl, G):
    """merge(shards) is exactly the top-k of the union of the shards' logits;
    against the oracle it passes the parity rules; the CUDA-core kernel's
    per-row arithmetic does not depend on the sharding, so there the merged
    result equals the single-GPU one bit-for-bit."""
    from paper_2605_26444_b200 import ActiveVocab, draft_logits_topk, merge_topk
    from paper_2605_26444_b200._native import NanoSpecError, EUNSUPPORTED
    V, d, W_max, n, k = 40000, 1024, 8192, 60, 10
    W = SI.bf16_weights(V, d, seed=7, device="cuda")
    z = SI.Zipf(V)
    p, pre = SI.prompt_and_prefill(z, 4, 3000, 3)
    pt = torch.as_tensor(p, device="cuda")
    prt = torch.as_tensor(pre, device="cuda")
    H = SI.bf16_hidden(n, d, seed=8, device="cuda")
    full = ActiveVocab(V, W_max)
    full.init(0, pt, prt)
    try:
        v1, i1, l1, _ = draft_logits_topk(full, W, H.reshape(1, n, d), k, impl=impl)
    except NanoSpecError as e:
        if e.status == EUNSUPPORTED:
            pytest.skip("tensor-core head not built for this shape")
        raise
    cl, ci, cls, zs, idss = [], [], [], [], []
    for r in range(G):
        st = ActiveVocab(V, W_max, shard_rank=r, n_shards=G)
        st.init(0, pt, prt)
        Wr = W[r::G].contiguous()
        v, i, l, zz = draft_logits_topk(st, Wr, H.reshape(1, n, d), k, impl=impl, debug_logits=True)
        ids_r = st.read(0)["slots"]
        cl.append(v[0].clone())
        ci.append(i[0].clone())
        cls.append(l[0].clone())
        zs.append(zz[0, :, : len(ids_r)].cpu().numpy().astype(np.float64))
        idss.append(ids_r)
    ml, mi, mlse = merge_topk(torch.stack(cl), torch.stack(ci), torch.stack(cls), k)
    torch.cuda.synchronize()
    # exactness of the merge itself: top-k of the union of the shard logits
    allz = np.concatenate(zs, axis=1)
    allid = np.concatenate(idss)
    order = np.argsort(allid, kind="stable")
    u_v, u_i = O.topk(allz[:, order], allid[order], k)
    assert np.array_equal(mi.cpu().numpy(), u_i)
    assert np.array_equal(ml.cpu().numpy().astype(np.float64), u_v)
    # parity against the oracle over the full active set
    ids = full.read(0)["ids"]
    assert np.array_equal(np.sort(allid), ids)
    z_ref, A = O.logits(SI.bf16_bits(W), SI.bf16_bits(H), ids)
    v_ref, id_ref = O.topk(z_ref, ids, k)
    check_topk(ml.cpu().numpy(), mi.cpu().numpy(), z_ref, A, ids, v_ref, id_ref, f"merged G={G}")
    check_lse(mlse.cpu().numpy(), O.lse(z_ref), "merged lse")
    if impl == "simt":
        assert torch.equal(mi, i1[0]) and torch.equal(ml, v1[0])
