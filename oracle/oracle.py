"""ctypes binding of the NanoSpec CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, ``__graft_entry__.smoke()``
and bench.py (its ``cpu_baseline`` leg and ``--impl reference``) may import this
module.  It shares nothing with the CUDA path in ``paper_2605_26444_b200/``.

Each wrapper cites the PAPER.md passage (P:n) its C function follows; the C file
header lists the readings of the paper it takes.  Marshalling only: all
arithmetic is in oracle.c.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

RULE_WINDOW = 0       # R1: Eq. 5 literally
RULE_UNIQUE_FIFO = 1  # R2: unique-FIFO reading


def build(force: bool = False) -> str:
    """Compile oracle.c with plain gcc -O2 (no intrinsics, no threads)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        i32p = ctypes.POINTER(ctypes.c_int32)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        u16p = ctypes.POINTER(ctypes.c_uint16)
        f64p = ctypes.POINTER(ctypes.c_double)
        L.oracle_bf16_to_double.argtypes = [ctypes.c_uint16]
        L.oracle_bf16_to_double.restype = ctypes.c_double
        L.oracle_stream_init.argtypes = [i32p, ctypes.c_int64, i32p, ctypes.c_int32, ctypes.c_int32, i32p, i32p]
        L.oracle_stream_init.restype = ctypes.c_int64
        L.oracle_stream_update.argtypes = [i32p, ctypes.c_int32, i32p, ctypes.c_int32, ctypes.c_int32, i32p, i32p]
        L.oracle_stream_update.restype = ctypes.c_int64
        L.oracle_active_set.argtypes = [i32p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                        ctypes.c_int32, ctypes.c_int32, i32p, u32p]
        L.oracle_active_set.restype = ctypes.c_int32
        L.oracle_ring.argtypes = [i32p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, i32p]
        L.oracle_ring.restype = ctypes.c_int64
        L.oracle_logits.argtypes = [u16p, ctypes.c_int64, ctypes.c_int32, u16p, ctypes.c_int32, i32p,
                                    ctypes.c_int32, f64p, f64p]
        L.oracle_logits.restype = None
        L.oracle_topk.argtypes = [f64p, i32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, f64p, i32p]
        L.oracle_topk.restype = None
        L.oracle_lse.argtypes = [f64p, ctypes.c_int32, ctypes.c_int32, f64p]
        L.oracle_lse.restype = None
        L.oracle_tree_expand.argtypes = [f64p, i32p, ctypes.c_int32, f64p, i32p, f64p, ctypes.c_int32, f64p, i32p,
                                         i32p, ctypes.c_int32, ctypes.c_int32, i32p, f64p]
        L.oracle_tree_expand.restype = None
        L.oracle_tree_rerank.argtypes = [f64p, ctypes.c_int32, ctypes.c_int32, i32p]
        L.oracle_tree_rerank.restype = None
        _lib = L
    return _lib


def _i32(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def _u16(a):
    a = np.ascontiguousarray(a, dtype=np.uint16)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint16))


def _f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class EmptyPrompt(ValueError):
    """Eq. 3 needs L >= 1 ("empty prompt")."""


def bf16_to_double(bits: int) -> float:
    return lib().oracle_bf16_to_double(int(bits) & 0xFFFF)


def stream_init(prompt, prefill_topk, vocab: int):
    """Eq. 3. prefill_topk: [L, k_pre] ids in rank order (or None).
    Returns (S0 as int32 array, err flag)."""
    prompt, pp = _i32(np.asarray(prompt).reshape(-1))
    L = prompt.size
    if prefill_topk is None:
        pre = np.zeros((L, 0), np.int32)
    else:
        pre = np.asarray(prefill_topk, np.int32).reshape(L, -1)
    k_pre = pre.shape[1]
    pre, ppre = _i32(pre.reshape(-1) if pre.size else np.zeros(1, np.int32))
    out = np.empty(L + L * k_pre + 1, np.int32)
    out, po = _i32(out)
    err = np.zeros(1, np.int32)
    err, pe = _i32(err)
    n = lib().oracle_stream_init(pp, L, ppre, k_pre, vocab, po, pe)
    if n < 0:
        raise EmptyPrompt("empty prompt")
    return out[:n].copy(), int(err[0])


def stream_update(draft, verify, vocab: int):
    """Eq. 4: the segment tuple(C_draft) (+) tuple(C_ver).
    Returns (segment, err flag)."""
    draft = np.asarray(draft if draft is not None else [], np.int32).reshape(-1)
    verify = np.asarray(verify if verify is not None else [], np.int32).reshape(-1)
    d, pd = _i32(draft if draft.size else np.zeros(1, np.int32))
    v, pv = _i32(verify if verify.size else np.zeros(1, np.int32))
    out, po = _i32(np.empty(draft.size + verify.size + 1, np.int32))
    err, pe = _i32(np.zeros(1, np.int32))
    n = lib().oracle_stream_update(pd, draft.size, pv, verify.size, vocab, po, pe)
    return out[:n].copy(), int(err[0])


def active_set(stream, vocab: int, w_max: int, rule: int = RULE_WINDOW, shard_rank: int = 0, n_shards: int = 1):
    """Eq. 5 (rule R1) or unique-FIFO (rule R2).
    Returns (ids ascending int32, bitmap uint32[ceil(V_local/32)])."""
    S, ps = _i32(np.asarray(stream, np.int32).reshape(-1) if len(stream) else np.zeros(1, np.int32))
    n_local = (vocab - shard_rank + n_shards - 1) // n_shards if n_shards > 1 else vocab
    ids, pi = _i32(np.empty(max(vocab, 1), np.int32))
    bm = np.zeros((n_local + 31) // 32, np.uint32)
    pb = bm.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))
    n = lib().oracle_active_set(ps, len(stream), vocab, w_max, rule, shard_rank, n_shards, pi, pb)
    return ids[:n].copy(), bm


def ring(stream, vocab: int, w_max: int, rule: int = RULE_WINDOW):
    """The W_max-slot ring of a GPU-resident state and its `total` counter."""
    S, ps = _i32(np.asarray(stream, np.int32).reshape(-1) if len(stream) else np.zeros(1, np.int32))
    r, pr = _i32(np.empty(w_max, np.int32))
    total = lib().oracle_ring(ps, len(stream), vocab, w_max, rule, pr)
    return r, int(total)


def logits(W_bits, H_bits, ids, want_abs: bool = True):
    """Eq. 2 restricted to I, fp64.  W_bits: uint16 [V, ldw] (bf16 bit
    patterns, only the first d columns used); H_bits: uint16 [n, d].
    Returns (z [n, |I|], A [n, |I|] or None)."""
    W_bits = np.asarray(W_bits)
    H_bits = np.asarray(H_bits)
    n, d = H_bits.shape
    ldw = W_bits.shape[1]
    W, pw = _u16(W_bits)
    H, ph = _u16(H_bits)
    ids = np.asarray(ids, np.int32).reshape(-1)
    m = int(ids.size)
    ids, pi = _i32(ids if m else np.zeros(1, np.int32))
    z, pz = _f64(np.empty((n, max(m, 1))))
    if want_abs:
        A, pa = _f64(np.empty((n, max(m, 1))))
    else:
        A, pa = None, None
    lib().oracle_logits(pw, ldw, d, ph, n, pi, m, pz, pa)
    return z[:, :m].copy(), (A[:, :m].copy() if want_abs else None)


def topk(z, ids, k: int):
    """SelectDraftTokens (Alg. 1): per row, (value desc, id asc) top-k,
    padded with (-inf, -1).  Returns (values f64 [n, k], ids int32 [n, k])."""
    z = np.asarray(z, np.float64)
    n, m = z.shape
    zz, pz = _f64(z if m else np.zeros((n, 1)))
    ii, pi = _i32(np.asarray(ids, np.int32).reshape(-1) if m else np.zeros(1, np.int32))
    v, pv = _f64(np.empty((n, k)))
    o, po = _i32(np.empty((n, k), np.int32))
    lib().oracle_topk(pz, pi, m, n, k, pv, po)
    return v, o


def lse(z):
    """log-sum-exp over the active set, fp64.  Returns [n]."""
    z = np.asarray(z, np.float64)
    n, m = z.shape
    zz, pz = _f64(z if m else np.zeros((n, 1)))
    out, po = _f64(np.empty(n))
    lib().oracle_lse(pz, m, n, po)
    return out


class OracleTree:
    """EAGLE-2 draft-tree node pool (Alg. 1; log-softmax over I,
    P:337): expand() one level from the head's top-k / lse of the frontier,
    rerank() the best m nodes.  Marshalling only (oracle.c does the arithmetic)."""

    def __init__(self, cap: int):
        self.score = np.full(cap, -np.inf)
        self.id = np.full(cap, -1, np.int32)
        self.parent = np.full(cap, -1, np.int32)
        self.n = 0
        self.front_index = None
        self.front_score = None

    def expand(self, val, ids, lse, n_next: int, front_score=None, front_index=None):
        val = np.ascontiguousarray(np.asarray(val, np.float64))
        n_front, k = val.shape
        ids_, pi = _i32(np.asarray(ids, np.int32).reshape(-1))
        v_, pv = _f64(val)
        l_, pl = _f64(np.asarray(lse, np.float64).reshape(-1))
        fs = self.front_score if front_score is None else np.asarray(front_score, np.float64)
        fi = self.front_index if front_index is None else np.asarray(front_index, np.int32)
        root = self.n == 0
        fs_, pfs = (None, None) if root else _f64(fs)
        fi_, pfi = (None, None) if root else _i32(fi)
        ps_, pps = _f64(self.score)
        pid_, ppid = _i32(self.id)
        ppar_, pppar = _i32(self.parent)
        ni_, pni = _i32(np.zeros(max(n_next, 1), np.int32))
        ns_, pns = _f64(np.zeros(max(n_next, 1)))
        lib().oracle_tree_expand(pfs, pfi, n_front, pv, pi, pl, k, pps, ppid, pppar, self.n, n_next, pni, pns)
        self.score, self.id, self.parent = ps_, pid_, ppar_
        self.n += n_front * k
        self.front_index, self.front_score = ni_[:n_next].copy(), ns_[:n_next].copy()
        return self.front_index, self.front_score

    def rerank(self, m: int):
        s_, ps = _f64(self.score[: self.n].copy())
        o_, po = _i32(np.zeros(m, np.int32))
        lib().oracle_tree_rerank(ps, self.n, m, po)
        return o_.copy(), self.id[o_].copy()


class OracleStream:
    """The whole candidate stream S kept on the host (no window truncation), with
    the active set recomputed from scratch by Eq. 5 on every read."""

    def __init__(self, vocab: int, w_max: int, rule: int = RULE_WINDOW):
        self.vocab, self.w_max, self.rule = vocab, w_max, rule
        self.S = np.zeros(0, np.int32)
        self.err = 0

    def init(self, prompt, prefill_topk=None):
        s, e = stream_init(prompt, prefill_topk, self.vocab)
        self.S, self.err = s, e
        return self

    def update(self, draft, verify):
        seg, e = stream_update(draft, verify, self.vocab)
        self.S = np.concatenate([self.S, seg])
        self.err |= e
        return self

    def active(self, shard_rank: int = 0, n_shards: int = 1):
        return active_set(self.S, self.vocab, self.w_max, self.rule, shard_rank, n_shards)

    def ring(self):
        return ring(self.S, self.vocab, self.w_max, self.rule)
