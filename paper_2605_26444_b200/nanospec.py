"""Thin Python binding over the C ABI (include/nanospec.h).

Argument marshalling only: torch provides device memory and the current CUDA
stream; every step of the path runs in the library's kernels.  Function names
follow the ABI (and the paper's notation).
"""
from __future__ import annotations

import ctypes

import torch

from . import _native as N

RULES = {"window": 0, "unique_fifo": 1}
IMPLS = {"auto": 0, "simt": 1, "tc": 2}


def _stream(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _need(t, dtype, name, device=None, numel=None):
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name} must have {numel} elements, got {t.numel()}")
    return t


def state_workspace_bytes(vocab, w_max, batch=1, rule="window", shard_rank=0, n_shards=1) -> int:
    return int(N.lib().nanospec_state_workspace_bytes(vocab, w_max, batch, RULES[rule], shard_rank, n_shards))


def head_scratch_bytes(batch, max_ids, n_nodes) -> int:
    return int(N.lib().nanospec_head_scratch_bytes(batch, max_ids, n_nodes))


class ActiveVocab:
    """GPU-resident candidate-stream state for `batch` sequences (a1/a2).

    I = Unique(Suffix(S, W_max)) (Eq. 5) kept as a bitmap + a stable
    slot table of ids entirely in device memory."""

    def __init__(self, vocab: int, w_max: int, batch: int = 1, rule: str = "window", shard_rank: int = 0,
                 n_shards: int = 1, device=None):
        self.vocab, self.w_max, self.batch, self.rule = vocab, w_max, batch, rule
        self.shard_rank, self.n_shards = shard_rank, n_shards
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        nbytes = state_workspace_bytes(vocab, w_max, batch, rule, shard_rank, n_shards)
        if nbytes == 0:
            raise N.NanoSpecError(N.EINVAL, "nanospec_state_workspace_bytes")
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        off = (-self.workspace.data_ptr()) % 256
        self._ws_ptr = self.workspace.data_ptr() + off
        self._ws_bytes = nbytes
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            N.check(N.lib().nanospec_state_create(ctypes.byref(h), vocab, w_max, batch, RULES[rule], shard_rank,
                                                  n_shards, self._ws_ptr, nbytes, _stream(self.device)),
                    "nanospec_state_create")
        self.handle = h.value
        self.v_local = (vocab - shard_rank + n_shards - 1) // n_shards if n_shards > 1 else vocab
        self.words = (self.v_local + 31) // 32

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                N.lib().nanospec_state_destroy(h)
            except Exception:
                pass
            self.handle = None

    # a1: Eq. 3
    def init(self, seq: int, prompt: torch.Tensor, prefill_topk: torch.Tensor | None = None):
        _need(prompt, torch.int32, "prompt")
        k_pre = 0
        if prefill_topk is not None:
            _need(prefill_topk, torch.int32, "prefill_topk")
            L = prompt.numel()
            if prefill_topk.numel() % max(L, 1):
                raise ValueError("prefill_topk must be [L, k_pre]")
            k_pre = prefill_topk.numel() // L if L else 0
        st = N.lib().nanospec_state_init(self.handle, seq, _ptr(prompt), prompt.numel(),
                                         _ptr(prefill_topk) if k_pre else None, k_pre, _stream(self.device))
        N.check(st, "nanospec_state_init")

    # a2: Eq. 4 + Eq. 5
    def update(self, seq: int, draft: torch.Tensor | None, verify: torch.Tensor | None):
        nd = 0 if draft is None else _need(draft, torch.int32, "draft").numel()
        kv = 0 if verify is None else _need(verify, torch.int32, "verify").numel()
        N.check(N.lib().nanospec_state_update(self.handle, seq, _ptr(draft) if nd else None, nd,
                                              _ptr(verify) if kv else None, kv, _stream(self.device)),
                "nanospec_state_update")

    def update_batch(self, draft: torch.Tensor | None, verify: torch.Tensor | None):
        nd = 0 if draft is None else _need(draft, torch.int32, "draft").numel() // self.batch
        kv = 0 if verify is None else _need(verify, torch.int32, "verify").numel() // self.batch
        N.check(N.lib().nanospec_state_update_batch(self.handle, _ptr(draft) if nd else None, nd,
                                                    _ptr(verify) if kv else None, kv, _stream(self.device)),
                "nanospec_state_update_batch")

    def read(self, seq: int) -> dict:
        """Synchronises the current stream; host copies of sequence `seq`'s state.
        `ids` is I in canonical ascending order, `slots` the device slot table
        (the row order of the head's debug logits)."""
        import numpy as np
        ids = np.empty(self.w_max, np.int32)
        bm = np.empty(self.words, np.uint32)
        ring = np.empty(self.w_max, np.int32)
        n = ctypes.c_int32()
        total = ctypes.c_int64()
        err = ctypes.c_int32()
        N.check(N.lib().nanospec_state_read(self.handle, seq, ids.ctypes.data, ctypes.byref(n), bm.ctypes.data,
                                            ring.ctypes.data, ctypes.byref(total), ctypes.byref(err),
                                            _stream(self.device)), "nanospec_state_read")
        slots = ids[: n.value].copy()
        return dict(ids=np.sort(slots), slots=slots, n_active=n.value, bitmap=bm, ring=ring, total=total.value,
                    err=err.value)

    def check(self) -> int:
        """Synchronises; returns the status (OK or EDEVICE)."""
        st = N.lib().nanospec_state_check(self.handle, _stream(self.device))
        if st not in (N.OK, N.EDEVICE):
            N.check(st, "nanospec_state_check")
        return st

    def ids_ptr(self, seq: int) -> int:
        return N.lib().nanospec_state_ids_ptr(self.handle, seq)

    def n_active_ptr(self, seq: int) -> int:
        return N.lib().nanospec_state_n_active_ptr(self.handle, seq)


class HeadOutputs:
    """Preallocated outputs + scratch for repeated (graph-captured) head calls."""

    def __init__(self, batch: int, n_nodes: int, k: int, max_ids: int, device, lse: bool = True,
                 debug_logits: bool = False):
        self.batch, self.n_nodes, self.k, self.max_ids = batch, n_nodes, k, max_ids
        self.topk_logit = torch.empty(batch, n_nodes, k, dtype=torch.float32, device=device)
        self.topk_id = torch.empty(batch, n_nodes, k, dtype=torch.int32, device=device)
        self.lse = torch.empty(batch, n_nodes, dtype=torch.float32, device=device) if lse else None
        self.debug_logits = (torch.empty(batch, n_nodes, max_ids, dtype=torch.float32, device=device)
                             if debug_logits else None)
        nbytes = head_scratch_bytes(batch, max_ids, n_nodes)
        if nbytes == 0:
            raise N.NanoSpecError(N.EINVAL, "nanospec_head_scratch_bytes")
        self.scratch = torch.zeros(nbytes, dtype=torch.uint8, device=device)


def _check_out(out: HeadOutputs, batch: int, n_nodes: int, k: int, max_ids: int, debug: bool = False):
    """A caller-supplied HeadOutputs must match the call: the kernels write
    [batch, n_nodes, k] outputs and use a scratch sized for max_ids rows."""
    if out.batch != batch or out.n_nodes != n_nodes or out.k != k or out.max_ids < max_ids:
        raise ValueError(f"HeadOutputs(batch={out.batch}, n_nodes={out.n_nodes}, k={out.k}, max_ids={out.max_ids}) "
                         f"does not fit a call with batch={batch}, n_nodes={n_nodes}, k={k}, max_ids={max_ids}")
    if debug and out.debug_logits is None:
        raise ValueError("debug logits requested but the HeadOutputs has no debug buffer")


def draft_logits_topk(state: ActiveVocab, w_head: torch.Tensor, hidden: torch.Tensor, k: int, *,
                      lse: bool = True, debug_logits: bool = False, impl: str = "auto",
                      out: HeadOutputs | None = None):
    """a3+a4+a5: top-k over W_head[I] h for every sequence and node.

    hidden: bf16 [batch, n_nodes, d] (or [n_nodes, d] when batch == 1).
    Returns (topk_logit [B,n,k] fp32, topk_id [B,n,k] int32, lse [B,n] or None,
    debug_logits [B,n,W_max] or None)."""
    _need(w_head, torch.bfloat16, "w_head")
    _need(hidden, torch.bfloat16, "hidden")
    d = w_head.shape[-1]
    n_nodes = hidden.numel() // (state.batch * d)
    if hidden.numel() != state.batch * n_nodes * d or hidden.shape[-1] != d:
        raise ValueError("hidden must be [batch, n_nodes, d] with the weight's d")
    if out is None:
        out = HeadOutputs(state.batch, n_nodes, k, state.w_max, hidden.device, lse, debug_logits)
    _check_out(out, state.batch, n_nodes, k, state.w_max, debug_logits)
    st = N.lib().nanospec_draft_logits_topk_ex(
        state.handle, _ptr(w_head), d, w_head.stride(0), _ptr(hidden), n_nodes, k, _ptr(out.topk_logit),
        _ptr(out.topk_id), _ptr(out.lse), _ptr(out.debug_logits), _ptr(out.scratch), out.scratch.numel(),
        IMPLS[impl], _stream(hidden.device))
    N.check(st, "nanospec_draft_logits_topk")
    return out.topk_logit, out.topk_id, out.lse, out.debug_logits


def step(state: ActiveVocab, seq: int, draft: torch.Tensor | None, verify: torch.Tensor | None,
         w_head: torch.Tensor, hidden: torch.Tensor, k: int, *, lse: bool = True, out: HeadOutputs | None = None):
    """One decode step of sequence `seq`: the state update (Eq. 4/5) and the head
    over the updated active set, fused into one launch when the
    shape allows (nanospec_step).  hidden: bf16 [n_nodes, d].
    Returns (topk_logit [1,n,k], topk_id [1,n,k], lse [1,n] or None)."""
    _need(w_head, torch.bfloat16, "w_head")
    _need(hidden, torch.bfloat16, "hidden")
    d = w_head.shape[-1]
    n_nodes = hidden.numel() // d
    for t, name in ((draft, "draft"), (verify, "verify")):
        if t is not None:
            _need(t, torch.int32, name)
    if out is None:
        out = HeadOutputs(1, n_nodes, k, state.w_max, hidden.device, lse, False)
    _check_out(out, 1, n_nodes, k, state.w_max)
    st = N.lib().nanospec_step(
        state.handle, seq, _ptr(draft), 0 if draft is None else draft.numel(), _ptr(verify),
        0 if verify is None else verify.numel(), _ptr(w_head), d, w_head.stride(0), _ptr(hidden), n_nodes, k,
        _ptr(out.topk_logit), _ptr(out.topk_id), _ptr(out.lse), _ptr(out.scratch), out.scratch.numel(),
        _stream(hidden.device))
    N.check(st, "nanospec_step")
    return out.topk_logit, out.topk_id, out.lse


def step_debug(state: ActiveVocab, seq: int, draft: torch.Tensor | None, verify: torch.Tensor | None,
               w_head: torch.Tensor, hidden: torch.Tensor, k: int, *, out: HeadOutputs | None = None):
    """step() in its fused launch, also returning the logits of every streamed
    row: [n_nodes, w_max + n_draft + k_ver] -- the pre-update slots, then the
    update-list entries (nanospec_step_debug).  Raises EUNSUPPORTED when the
    step cannot be fused."""
    _need(w_head, torch.bfloat16, "w_head")
    _need(hidden, torch.bfloat16, "hidden")
    d = w_head.shape[-1]
    n_nodes = hidden.numel() // d
    nd = 0 if draft is None else _need(draft, torch.int32, "draft").numel()
    kv = 0 if verify is None else _need(verify, torch.int32, "verify").numel()
    if out is None:
        out = HeadOutputs(1, n_nodes, k, state.w_max, hidden.device)
    _check_out(out, 1, n_nodes, k, state.w_max)
    dbg = torch.full((n_nodes, state.w_max + nd + kv), float("nan"), dtype=torch.float32, device=hidden.device)
    st = N.lib().nanospec_step_debug(
        state.handle, seq, _ptr(draft), nd, _ptr(verify), kv, _ptr(w_head), d, w_head.stride(0), _ptr(hidden), n_nodes,
        k, _ptr(out.topk_logit), _ptr(out.topk_id), _ptr(out.lse), _ptr(dbg), _ptr(out.scratch), out.scratch.numel(),
        _stream(hidden.device))
    N.check(st, "nanospec_step_debug")
    return out.topk_logit, out.topk_id, out.lse, dbg


class StepHostIO:
    """Device staging for nanospec_step_host (the end-to-end call with HOST
    buffers): pinned host blocks in the ABI's packed layouts
    in  = [hidden bf16 n x d][draft int32 n_draft][verify int32 k_ver],
    out = [topk_logit fp32 n x k][topk_id int32 n x k][lse fp32 n]."""

    def __init__(self, n_nodes: int, d_model: int, n_draft: int, k_ver: int, k: int, w_max: int, device,
                 slots: int = 1):
        """slots >= 2: a pipeline (nanospec_step_host_async) -- each step's input
        copy runs on a copy stream while the previous step computes; the slots'
        staging, host results and events alternate."""
        ib, ob = ctypes.c_size_t(0), ctypes.c_size_t(0)
        total = N.lib().nanospec_step_host_io_bytes(n_nodes, d_model, n_draft, k_ver, k, ctypes.byref(ib),
                                                    ctypes.byref(ob))
        if total == 0:
            raise N.NanoSpecError(N.EINVAL, "nanospec_step_host_io_bytes")
        self.n, self.d, self.n_draft, self.k_ver, self.k = n_nodes, d_model, n_draft, k_ver, k
        self.in_bytes, self.out_bytes = ib.value, ob.value
        self.slots = slots
        self.total = total
        self.d_ios = [torch.empty(total, dtype=torch.uint8, device=device) for _ in range(slots)]
        self.d_io = self.d_ios[0]
        self.scratch = HeadOutputs(1, n_nodes, k, w_max, device).scratch
        self.h_outs = [torch.empty(self.out_bytes, dtype=torch.uint8).pin_memory() for _ in range(slots)]
        self.h_out = self.h_outs[0]
        self.slot = 0  # the slot of the most recent step
        if slots > 1:
            self.copy_stream = torch.cuda.Stream(device)
            self.ev_in = [torch.cuda.Event() for _ in range(slots)]
            self.ev_done = [torch.cuda.Event() for _ in range(slots)]
            for e in self.ev_in + self.ev_done:  # create the events (torch creates them lazily)
                e.record(self.copy_stream)
            torch.cuda.current_stream(device).wait_stream(self.copy_stream)
        # input blocks handed to nanospec_step_host stay referenced until the
        # stream has consumed them (the library's cudaMemcpyAsync is invisible
        # to torch's pinned-memory allocator, which could otherwise recycle them)
        self._inflight = []

    def _retire(self):
        self._inflight = [(ev, blk) for ev, blk in self._inflight if not ev.query()]

    def pack_inputs(self, hidden: torch.Tensor, draft, verify) -> torch.Tensor:
        """A pinned host block holding one step's inputs."""
        self._retire()
        blk = torch.zeros(self.in_bytes, dtype=torch.uint8).pin_memory()
        hb = self.n * self.d * 2
        blk[:hb].view(torch.bfloat16).copy_(hidden.reshape(-1).cpu())
        blk[hb:hb + 4 * self.n_draft].view(torch.int32).copy_(torch.as_tensor(draft, dtype=torch.int32).cpu())
        blk[hb + 4 * self.n_draft:hb + 4 * (self.n_draft + self.k_ver)].view(torch.int32).copy_(
            torch.as_tensor(verify, dtype=torch.int32).cpu())
        return blk

    def results(self, slot: int | None = None):
        """(topk_logit [n,k], topk_id [n,k], lse [n]) views of a host result block
        (default: the most recent step's; a pipeline's step is complete once
        its ev_done event is)."""
        nk = self.n * self.k
        h = self.h_outs[self.slot if slot is None else slot]
        return (h[:4 * nk].view(torch.float32).view(self.n, self.k),
                h[4 * nk:8 * nk].view(torch.int32).view(self.n, self.k),
                h[8 * nk:8 * nk + 4 * self.n].view(torch.float32))


def step_host(state: ActiveVocab, seq: int, io: StepHostIO, h_in: torch.Tensor, w_head: torch.Tensor, k: int):
    """nanospec_step_host: H2D of the packed inputs, the step, D2H of the packed
    results, asynchronous on the current stream (results in io.results() after a sync)."""
    _need(w_head, torch.bfloat16, "w_head")
    if io.slots > 1:  # pipelined: the input copy on io.copy_stream, slots alternate
        sl = (io.slot + 1) % io.slots
        st = N.lib().nanospec_step_host_async(
            state.handle, seq, h_in.data_ptr(), io.n_draft, io.k_ver, _ptr(w_head), io.d, w_head.stride(0), io.n, k,
            io.h_outs[sl].data_ptr(), _ptr(io.d_ios[sl]), io.total, _ptr(io.scratch), io.scratch.numel(),
            _stream(w_head.device), io.copy_stream.cuda_stream, io.ev_in[sl].cuda_event, io.ev_done[sl].cuda_event)
        N.check(st, "nanospec_step_host_async")
        io.slot = sl
    else:
        st = N.lib().nanospec_step_host(
            state.handle, seq, h_in.data_ptr(), io.n_draft, io.k_ver, _ptr(w_head), io.d, w_head.stride(0), io.n, k,
            io.h_out.data_ptr(), _ptr(io.d_io), io.d_io.numel(), _ptr(io.scratch), io.scratch.numel(),
            _stream(w_head.device))
        N.check(st, "nanospec_step_host")
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream(w_head.device))
    io._inflight.append((ev, h_in))


def step_is_fused(state: ActiveVocab, n_draft: int, k_ver: int, d_model: int, n_nodes: int, k: int) -> bool:
    """Whether step() with these sizes runs as one fused launch on this device."""
    return bool(N.lib().nanospec_step_fused(state.handle, n_draft, k_ver, d_model, n_nodes, k))


def logits_topk_ids(ids: torch.Tensor, n_ids: torch.Tensor, w_head: torch.Tensor, hidden: torch.Tensor, k: int, *,
                    n_shards: int = 1, lse: bool = True, debug_logits: bool = False, impl: str = "auto",
                    out: HeadOutputs | None = None):
    """The head over an explicit ascending id list (e.g. [0, V): the dense
    full-vocabulary head of Eq. 2).  n_ids: int32 [1] on device."""
    _need(ids, torch.int32, "ids")
    _need(n_ids, torch.int32, "n_ids", numel=1)
    _need(w_head, torch.bfloat16, "w_head")
    _need(hidden, torch.bfloat16, "hidden")
    d = w_head.shape[-1]
    n_nodes = hidden.numel() // d
    if out is None:
        out = HeadOutputs(1, n_nodes, k, ids.numel(), hidden.device, lse, debug_logits)
    _check_out(out, 1, n_nodes, k, ids.numel(), debug_logits)
    st = N.lib().nanospec_logits_topk_ids(
        _ptr(ids), _ptr(n_ids), ids.numel(), n_shards, _ptr(w_head), d, w_head.stride(0), _ptr(hidden), n_nodes, k,
        _ptr(out.topk_logit), _ptr(out.topk_id), _ptr(out.lse), _ptr(out.debug_logits), _ptr(out.scratch),
        out.scratch.numel(), IMPLS[impl], _stream(hidden.device))
    N.check(st, "nanospec_logits_topk_ids")
    return out.topk_logit, out.topk_id, out.lse, out.debug_logits


def merge_topk(cand_logit: torch.Tensor, cand_id: torch.Tensor, cand_lse: torch.Tensor | None, k: int):
    """Exact top-k / lse over the union of vocab shards.
    cand_logit/cand_id: [S, rows, k]; cand_lse: [S, rows]."""
    _need(cand_logit, torch.float32, "cand_logit")
    _need(cand_id, torch.int32, "cand_id")
    S = cand_logit.shape[0]
    rows = cand_logit.numel() // (S * k)
    ol = torch.empty(rows, k, dtype=torch.float32, device=cand_logit.device)
    oi = torch.empty(rows, k, dtype=torch.int32, device=cand_logit.device)
    olse = None
    if cand_lse is not None:
        _need(cand_lse, torch.float32, "cand_lse")
        olse = torch.empty(rows, dtype=torch.float32, device=cand_logit.device)
    N.check(N.lib().nanospec_merge_topk(_ptr(cand_logit), _ptr(cand_id), _ptr(cand_lse), S, rows, k, _ptr(ol),
                                        _ptr(oi), _ptr(olse), _stream(cand_logit.device)), "nanospec_merge_topk")
    return ol, oi, olse


class DraftTree:
    """Device node pool of one EAGLE-2-style draft round (Alg. 1
    P:523-530; depth 5 and 60 draft tokens): expand() appends a level's
    children with cumulative log-probability scores (log-softmax over I,
    P:337) and picks the next frontier; rerank() keeps the best `m` nodes --
    their tokens are C_draft of the state update.  Fixed
    buffers, so a whole round can be captured in one CUDA graph."""

    def __init__(self, pool_cap: int, width: int, device):
        if not 1 <= pool_cap <= 4096:
            raise ValueError("pool_cap must be in [1, 4096]")
        self.cap, self.width = pool_cap, width
        self.score = torch.full((pool_cap,), float("-inf"), dtype=torch.float32, device=device)
        self.id = torch.full((pool_cap,), -1, dtype=torch.int32, device=device)
        self.parent = torch.full((pool_cap,), -1, dtype=torch.int32, device=device)
        self.front_index = torch.zeros(width, dtype=torch.int32, device=device)
        self.front_score = torch.zeros(width, dtype=torch.float32, device=device)
        self.n = 0
        self.n_front = 0

    def reset(self):
        self.n = 0
        self.n_front = 0

    def expand(self, topk_logit: torch.Tensor, topk_id: torch.Tensor, lse: torch.Tensor, n_next: int):
        """One level: the head outputs of the current frontier (root when the
        pool is empty) -> children in the pool, the best n_next as the frontier."""
        n_front, k = topk_logit.shape[-2], topk_logit.shape[-1]
        root = self.n == 0
        st = N.lib().nanospec_tree_expand(
            None if root else _ptr(self.front_score), None if root else _ptr(self.front_index), n_front,
            _ptr(topk_logit), _ptr(topk_id), _ptr(lse), k, _ptr(self.score), _ptr(self.id), _ptr(self.parent),
            self.n, self.cap, n_next, _ptr(self.front_index), _ptr(self.front_score), _stream(topk_logit.device))
        N.check(st, "nanospec_tree_expand")
        self.n += n_front * k
        self.n_front = n_next

    def rerank(self, m: int, out_index: torch.Tensor | None = None, out_id: torch.Tensor | None = None):
        """The m best nodes of the pool: (pool indices [m], token ids [m])."""
        dev = self.score.device
        out_index = torch.empty(m, dtype=torch.int32, device=dev) if out_index is None else out_index
        out_id = torch.empty(m, dtype=torch.int32, device=dev) if out_id is None else out_id
        N.check(N.lib().nanospec_tree_rerank(_ptr(self.score), _ptr(self.id), self.n, m, _ptr(out_index),
                                             _ptr(out_id), _stream(dev)), "nanospec_tree_rerank")
        return out_index, out_id


class PackedHead:
    """The paper's repack design (T6 P:451) as a measured variant:
    a dense [batch, w_max, d] copy of the active rows kept in slot order.
    refresh() copies the rows of slots whose id changed (nanospec_repack; run
    it on a copy stream after the update), head() runs the tensor-core head on
    the packed rows (nanospec_draft_logits_topk_packed)."""

    def __init__(self, state: ActiveVocab, d_model: int, device):
        self.state, self.d = state, d_model
        self.packed = torch.zeros(state.batch, state.w_max, d_model, dtype=torch.bfloat16, device=device)
        self.tags = torch.full((state.batch, state.w_max), -1, dtype=torch.int32, device=device)

    def refresh(self, seq: int, w_head: torch.Tensor):
        _need(w_head, torch.bfloat16, "w_head")
        N.check(N.lib().nanospec_repack(self.state.handle, seq, _ptr(w_head), self.d, w_head.stride(0),
                                        _ptr(self.packed), self.d, _ptr(self.tags), _stream(w_head.device)),
                "nanospec_repack")

    def head(self, hidden: torch.Tensor, k: int, out: HeadOutputs):
        _need(hidden, torch.bfloat16, "hidden")
        n_nodes = hidden.numel() // (self.state.batch * self.d)
        _check_out(out, self.state.batch, n_nodes, k, self.state.w_max)
        N.check(N.lib().nanospec_draft_logits_topk_packed(
            self.state.handle, _ptr(self.packed), self.d, self.d, _ptr(hidden), n_nodes, k, _ptr(out.topk_logit),
            _ptr(out.topk_id), _ptr(out.lse), _ptr(out.scratch), out.scratch.numel(), _stream(hidden.device)),
            "nanospec_draft_logits_topk_packed")
        return out.topk_logit, out.topk_id, out.lse
