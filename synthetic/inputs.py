"""Seeded synthetic input generators shared by tests, bench.py and smoke().

This module holds NONE of the method's arithmetic (no stream rule, no
contraction, no top-k): it only draws token ids and tensors.  Both the CUDA path
and the CPU oracle consume what it returns, so neither side sees the other's
output.  Recipes:

* token streams: Zipf(s) over V ranks, P(rank r) ~ r^-s (s = 1.0 default),
  mapped to token ids through a seeded permutation so that frequent tokens are
  not clustered by id;
* draft tree tokens: 60 Zipf draws per step (an EAGLE-2 60-node tree),
  duplicates allowed -- the state dedups them (tuple(C_draft));
* verify candidates: K_ver = 3 distinct Zipf draws (T_Kver returns distinct ids);
* prefill candidates: [L, K_pre] distinct-per-row Zipf draws;
* LM-head weight W ~ bf16(N(0, 0.02^2)), hidden states H ~ bf16(N(0, 1)).
"""
from __future__ import annotations

import numpy as np

try:  # torch is only needed for the tensor generators
    import torch
except Exception:  # pragma: no cover
    torch = None


LLAMA = dict(name="llama-3.1-8b", vocab=128256, d_model=4096)
QWEN = dict(name="qwen-2.5-7b", vocab=152064, d_model=3584)
TINY = dict(name="tiny", vocab=1000, d_model=64)


class Zipf:
    """Zipf(s) over `vocab` ranks with a seeded rank->id permutation."""

    def __init__(self, vocab: int, s: float = 1.0, perm_seed: int = 3, identity: bool = False):
        self.vocab = vocab
        ranks = np.arange(1, vocab + 1, dtype=np.float64)
        p = ranks ** (-s)
        self.cdf = np.cumsum(p / p.sum())
        self.cdf[-1] = 1.0
        self.perm = (np.arange(vocab, dtype=np.int64) if identity
                     else np.random.default_rng(perm_seed).permutation(vocab))

    def draw(self, rng: np.random.Generator, n: int) -> np.ndarray:
        r = np.searchsorted(self.cdf, rng.random(n), side="right")
        return self.perm[np.minimum(r, self.vocab - 1)].astype(np.int32)

    def draw_distinct(self, rng: np.random.Generator, n: int) -> np.ndarray:
        out: list[int] = []
        seen: set[int] = set()
        while len(out) < n:
            for t in self.draw(rng, 2 * n):
                t = int(t)
                if t not in seen:
                    seen.add(t)
                    out.append(t)
                    if len(out) == n:
                        break
        return np.asarray(out, np.int32)


def prompt_and_prefill(zipf: Zipf, seed: int, L: int, k_pre: int):
    """A Zipf prompt x_1..x_L and a [L, k_pre] table of per-position candidates."""
    rng = np.random.default_rng(seed)
    prompt = zipf.draw(rng, L)
    pre = np.stack([zipf.draw_distinct(rng, k_pre) for _ in range(L)]) if k_pre else np.zeros((L, 0), np.int32)
    return prompt, pre.astype(np.int32)


def decode_steps(zipf: Zipf, seed: int, steps: int, n_draft: int = 60, k_ver: int = 3):
    """`steps` update batches (draft tree tokens, verify top-k)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(steps):
        out.append((zipf.draw(rng, n_draft), zipf.draw_distinct(rng, k_ver)))
    return out


def disjoint_pools(vocab: int, pool: int, count: int, seed: int = 3) -> np.ndarray:
    """`count` pairwise-disjoint id pools of size `pool` (a seeded permutation cut
    into pieces); used to rotate cold active sets through the bench."""
    assert pool * count <= vocab, (pool, count, vocab)
    perm = np.random.default_rng(seed).permutation(vocab).astype(np.int32)
    return perm[: pool * count].reshape(count, pool)


def cyclic_fresh_updates(pool_ids: np.ndarray, w_max: int, steps: int, n_draft: int = 60, k_ver: int = 3):
    """Headline |I| = W_max recipe: the prompt is the first w_max ids of the pool
    (all distinct); each step appends the next n_draft + k_ver ids of the pool in
    cyclic order.  With len(pool) >= w_max + n_draft + k_ver every appended id is
    outside the current window, so |I| stays exactly w_max."""
    P = len(pool_ids)
    m = n_draft + k_ver
    assert P >= w_max + m
    prompt = pool_ids[:w_max].copy()
    ups = []
    pos = w_max
    for _ in range(steps):
        idx = (pos + np.arange(m)) % P
        seg = pool_ids[idx]
        ups.append((seg[:n_draft].copy(), seg[n_draft:].copy()))
        pos = (pos + m) % P
    return prompt, ups


def bf16_weights(vocab: int, d: int, seed: int = 0, device="cpu", std: float = 0.02):
    """W ~ bf16(N(0, std^2)), [vocab, d]."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return (torch.randn(vocab, d, generator=g, device=device) * std).to(torch.bfloat16)


def bf16_hidden(n: int, d: int, seed: int = 1, device="cpu", batch: int | None = None):
    """H ~ bf16(N(0, 1)), [n, d] or [batch, n, d]."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    shape = (n, d) if batch is None else (batch, n, d)
    return torch.randn(*shape, generator=g, device=device).to(torch.bfloat16)


def int_valued_bf16(shape, lo: int, hi: int, seed: int, device="cpu"):
    """Small integers stored exactly in bf16 (for order-independent exact sums)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return torch.randint(lo, hi + 1, shape, generator=g, device=device).to(torch.bfloat16)


def bf16_bits(t) -> np.ndarray:
    """The uint16 bit patterns of a bf16 tensor, as a host numpy array."""
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)
