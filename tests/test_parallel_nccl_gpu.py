"""Two ranks over NCCL on two GPUs: the vocab-parallel head
(cyclic row shards, one all-gather of the per-shard top-k + lse, exact merge)
and the data-parallel split of a batch, both against the oracle.  Skips on a
box with fewer than two GPUs (the gloo tests cover the host logic on CPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _vp_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        import paper_2605_26444_b200 as P
        from paper_2605_26444_b200 import parallel as PAR
        from synthetic import inputs as SI
        V, d, Wm, n, k = 20000, 512, 4096, 16, 10
        W = SI.bf16_weights(V, d, seed=0, device=dev)
        Wl = PAR.shard_rows_cyclic(W, rank, world)
        z = SI.Zipf(V)
        prompt, pre = SI.prompt_and_prefill(z, 3, 3000, 3)
        st = P.ActiveVocab(V, Wm, shard_rank=rank, n_shards=world, device=dev)
        st.init(0, torch.as_tensor(prompt, device=dev), torch.as_tensor(pre, device=dev))
        for dd, vv in SI.decode_steps(z, 4, 3):
            st.update(0, torch.as_tensor(dd, device=dev), torch.as_tensor(vv, device=dev))
        H = SI.bf16_hidden(n, d, seed=5, device=dev)
        v, i, l = PAR.vp_draft_logits_topk(st, Wl, H.reshape(1, n, d), k)
        torch.cuda.synchronize()
        q.put((rank, v.cpu().numpy(), i.cpu().numpy(), l.cpu().numpy()))
    except Exception as e:  # surfaced by the parent
        q.put((rank, repr(e), None, None))
    finally:
        dist.destroy_process_group()


def test_vocab_parallel_two_ranks_nccl(cuda_ok):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (one process per GPU over NCCL)")
    from oracle import oracle as O
    from synthetic import inputs as SI
    from parity import check_lse, check_topk
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_vp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(2):
        r, v, i, l = q.get(timeout=600)
        res[r] = (v, i, l)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert not isinstance(res[r][0], str), res[r][0]
    # replicated result, equal on both ranks
    assert np.array_equal(res[0][1], res[1][1]) and np.array_equal(res[0][0], res[1][0])
    V, d, Wm, n, k = 20000, 512, 4096, 16, 10
    z = SI.Zipf(V)
    prompt, pre = SI.prompt_and_prefill(z, 3, 3000, 3)
    ref = O.OracleStream(V, Wm).init(prompt, pre)
    for dd, vv in SI.decode_steps(z, 4, 3):
        ref.update(dd, vv)
    ids, _ = ref.active()
    Wb = SI.bf16_bits(SI.bf16_weights(V, d, seed=0))
    Hb = SI.bf16_bits(SI.bf16_hidden(n, d, seed=5))
    z_ref, A = O.logits(Wb, Hb, ids)
    v_ref, id_ref = O.topk(z_ref, ids, k)
    check_topk(res[0][0], res[0][1], z_ref, A, ids, v_ref, id_ref, "vp2 nccl")
    check_lse(res[0][2], O.lse(z_ref), "vp2 nccl")
