"""Host-side multi-GPU logic on CPU with gloo, world size 2.

* DP: dp_sequences partitions the sequences exactly.
* VP: cyclic row sharding; every rank's oracle shard of I; the candidate
  all-gather (pack -> collective -> unpack) returns every rank's candidates in
  rank order; the top-k of the gathered union equals the unsharded top-k
  (the property the GPU merge relies on)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_26444_b200 import parallel as PAR


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_dp_sequences_partition():
    for n in (1, 7, 64, 65):
        for w in (1, 2, 3, 8):
            got = [i for r in range(w) for i in PAR.dp_sequences(n, r, w)]
            assert got == list(range(n))
            sizes = [len(PAR.dp_sequences(n, r, w)) for r in range(w)]
            assert max(sizes) - min(sizes) <= 1


def test_shard_rows_cyclic():
    W = torch.arange(30).reshape(10, 3)
    for G in (2, 3):
        for r in range(G):
            S = PAR.shard_rows_cyclic(W, r, G)
            for l in range(S.shape[0]):
                assert torch.equal(S[l], W[l * G + r])


def test_pack_unpack_roundtrip():
    v = torch.randn(5, 4)
    i = torch.randint(-1, 1000, (5, 4), dtype=torch.int32)
    l = torch.randn(5)
    buf = PAR.pack_candidates(v, i, l)
    v2, i2, l2 = PAR.unpack_candidates(torch.cat([buf, buf]), 2, 5, 4)
    for w in range(2):
        assert torch.equal(v2[w], v) and torch.equal(i2[w], i) and torch.equal(l2[w], l)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from synthetic import inputs as SI
        V, d, Wm, n, k = 3000, 32, 700, 6, 10
        z = SI.Zipf(V)
        p, pre = SI.prompt_and_prefill(z, 4, 500, 3)
        ref = O.OracleStream(V, Wm).init(p, pre)
        for dd, vv in SI.decode_steps(z, 5, 8):
            ref.update(dd, vv)
        W = SI.bf16_weights(V, d, seed=3)
        H = SI.bf16_hidden(n, d, seed=4)
        ids, _ = ref.active(rank, world)
        Wl = PAR.shard_rows_cyclic(W, rank, world)
        # local rows g // world of the shard are the global rows g
        assert all(torch.equal(Wl[int(g) // world], W[int(g)]) for g in ids[:20])
        zl, _ = O.logits(SI.bf16_bits(W), SI.bf16_bits(H), ids)
        v, i = O.topk(zl, ids, k)
        l = O.lse(zl)
        cl, ci, cls = PAR.gather_candidates(torch.tensor(v, dtype=torch.float32), torch.tensor(i),
                                            torch.tensor(l, dtype=torch.float32))
        # union of shard candidates -> exact global top-k (up to fp32 rounding of the packed values)
        allv = cl.permute(1, 0, 2).reshape(n, -1).double().numpy()
        alli = ci.permute(1, 0, 2).reshape(n, -1).numpy()
        full_ids, _ = ref.active()
        zf, _ = O.logits(SI.bf16_bits(W), SI.bf16_bits(H), full_ids)
        vf, idf = O.topk(zf, full_ids, k)
        for row in range(n):
            order = np.lexsort((alli[row], -allv[row]))
            got = [int(alli[row][o]) for o in order if alli[row][o] >= 0][:k]
            assert got == idf[row].tolist()
        lse_all = np.logaddexp.reduce(cls.double().numpy(), axis=0)
        assert np.allclose(lse_all, O.lse(zf), rtol=1e-6)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_vp_gather_and_union_topk_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, "ok"), (1, "ok")], res
