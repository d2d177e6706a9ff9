"""Multi-GPU plumbing of the hot path; one process per GPU.

* Data parallel (DP): sequences are independent; rank r owns a contiguous block
  of them and runs the whole path locally.  No collective on the path.
* Vocab parallel (VP): rows of W_head are sharded cyclically (rank r owns ids
  g with g % G == r, stored at local row g // G); every rank applies the same
  update lists to its state shard (replicated ring, sharded bitmap/ids), runs
  the head on its rows, and the per-shard top-k (+ lse) meet in ONE NCCL
  all-gather, after which nanospec_merge_topk gives every rank the exact
  global result.

torch.distributed is used for the process group and the collective only.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def dp_sequences(n_seq: int, rank: int, world: int) -> range:
    """Contiguous, balanced block of sequence indices owned by `rank`."""
    base, extra = divmod(n_seq, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def shard_rows_cyclic(w_head: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    """Rows g with g % world == rank, at local row g // world."""
    return w_head[rank::world].contiguous()


def pack_candidates(topk_logit: torch.Tensor, topk_id: torch.Tensor, lse: torch.Tensor) -> torch.Tensor:
    """One fp32 buffer [n*k (logits) | n*k (ids, bit-cast) | n (lse)] so the
    exchange is a single collective."""
    return torch.cat([topk_logit.reshape(-1).float(), topk_id.reshape(-1).contiguous().view(torch.float32),
                      lse.reshape(-1).float()])


def unpack_candidates(buf: torch.Tensor, world: int, n: int, k: int):
    """[world, n*k*2 + n] -> (logit [world, n, k], id [world, n, k], lse [world, n])."""
    buf = buf.reshape(world, 2 * n * k + n)
    logit = buf[:, : n * k].reshape(world, n, k).contiguous()
    ids = buf[:, n * k: 2 * n * k].contiguous().view(torch.int32).reshape(world, n, k)
    lse = buf[:, 2 * n * k:].contiguous()
    return logit, ids, lse


def gather_candidates(topk_logit, topk_id, lse, group=None):
    """All-gather every rank's per-shard top-k + lse (NCCL over NVLink on GPUs;
    gloo on CPU for the host-logic tests)."""
    world = dist.get_world_size(group)
    n, k = topk_logit.shape[-2], topk_logit.shape[-1]
    mine = pack_candidates(topk_logit, topk_id, lse)
    out = torch.empty(world * mine.numel(), dtype=mine.dtype, device=mine.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, mine, group=group)
    else:
        parts = list(out.chunk(world))
        dist.all_gather(parts, mine, group=group)
        out = torch.cat(parts)
    return unpack_candidates(out, world, n, k)


def vp_draft_logits_topk(state, w_shard: torch.Tensor, hidden: torch.Tensor, k: int, *, group=None,
                         impl: str = "auto", out=None):
    """Vocab-parallel head: local head on this rank's rows, one all-gather of
    the candidates, exact merge.  Returns (topk_logit [n,k], topk_id [n,k],
    lse [n]) replicated on every rank."""
    from .nanospec import draft_logits_topk, merge_topk
    v, i, l, _ = draft_logits_topk(state, w_shard, hidden, k, impl=impl, out=out)
    cl, ci, cls = gather_candidates(v[0], i[0], l[0], group)
    return merge_topk(cl, ci, cls, k)
