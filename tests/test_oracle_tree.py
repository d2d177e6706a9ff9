"""Pins of the oracle's draft-tree bookkeeping (oracle.c: oracle_tree_expand /
oracle_tree_rerank; EAGLE-2 SelectDraftTokens, Alg. 1, depth 5 / 60
draft tokens P:286, log-softmax over the active set P:337), against things
fixed independently of it: a hand-worked two-level example in closed form,
the path-sum identity (a node's score is the sum of its ancestors' log-softmax
terms, recomputed by walking parents), brute-force sorting for the frontier
and the rerank, and the score-monotonicity invariant."""
import math

import numpy as np

from oracle import oracle as O


def test_hand_worked_two_levels():
    # active set of 3 tokens: root logits over I: token 10 -> 2, 11 -> 1, 12 -> 0
    lse0 = math.log(math.exp(2) + math.exp(1) + math.exp(0))
    t = O.OracleTree(16)
    fi, fs = t.expand([[2.0, 1.0]], [[10, 11]], [lse0], n_next=1)
    assert t.n == 2 and list(t.id[:2]) == [10, 11] and list(t.parent[:2]) == [-1, -1]
    assert abs(t.score[0] - (2 - lse0)) < 1e-15 and abs(t.score[1] - (1 - lse0)) < 1e-15
    assert list(fi) == [0] and abs(fs[0] - math.log(math.exp(2) / (math.exp(2) + math.exp(1) + 1))) < 1e-15
    # level 2 from node 0 (token 10): logits 0.5 / -0.5 for tokens 12 / 10, lse over I = log(e^.5 + e^-.5 + e^0)
    lse1 = math.log(math.exp(0.5) + math.exp(-0.5) + 1.0)
    fi2, fs2 = t.expand([[0.5, -0.5]], [[12, 10]], [lse1], n_next=2)
    want = [(2 - lse0) + (0.5 - lse1), (2 - lse0) + (-0.5 - lse1)]
    assert abs(t.score[2] - want[0]) < 1e-14 and abs(t.score[3] - want[1]) < 1e-14
    assert list(t.parent[2:4]) == [0, 0] and list(fi2) == [2, 3]
    # rerank over the whole pool: node 0 (-0.41), node 1 (-1.41), node 2, node 3
    idx, ids = t.rerank(3)
    order = sorted(range(4), key=lambda c: (-t.score[c], c))[:3]
    assert list(idx) == order and list(ids) == [int(t.id[c]) for c in order]


def _random_round(seed, k=10, width=10, depth=6, vocab=500):
    rng = np.random.default_rng(seed)
    t = O.OracleTree(1 + k + (depth - 1) * width * k + 8)
    term = {}  # pool node -> its own log-softmax term (val - lse)
    n_front = 1
    for d in range(depth):
        val = rng.normal(0, 2, (n_front, k))
        val = -np.sort(-val, axis=1)  # the head returns its top-k sorted
        ids = rng.integers(0, vocab, (n_front, k)).astype(np.int32)
        lse = val.max(axis=1) + rng.uniform(0.5, 3.0, n_front)  # lse over I exceeds every member
        base = t.n
        fi, fs = t.expand(val, ids, lse, n_next=width)
        for f in range(n_front):
            for j in range(k):
                term[base + f * k + j] = val[f, j] - lse[f]
        # frontier = the width best children of this level by (score desc, index asc)
        lvl = np.arange(base, t.n)
        order = lvl[np.lexsort((lvl, -t.score[lvl]))][:width]
        assert np.array_equal(fi, order)
        assert np.array_equal(fs, t.score[order])
        n_front = width
    return t, term


def test_path_sums_and_order():
    t, term = _random_round(3)
    for c in range(t.n):
        s, node = 0.0, c
        while node >= 0:
            s += term[node]
            node = int(t.parent[node])
        assert abs(t.score[c] - s) < 1e-12
        if t.parent[c] >= 0:  # log-probabilities only decrease along a path
            assert t.score[c] < t.score[int(t.parent[c])]
    idx, ids = t.rerank(60)
    allc = np.arange(t.n)
    want = allc[np.lexsort((allc, -t.score[: t.n]))][:60]
    assert np.array_equal(idx, want) and np.array_equal(ids, t.id[want])


def test_ties_and_padding():
    t = O.OracleTree(8)
    # two equal children: the lower pool index first; a padding child (-1) scores -inf and ranks last
    fi, fs = t.expand([[1.0, 1.0, 0.0]], [[7, 8, -1]], [2.0], n_next=3)
    assert list(fi) == [0, 1, 2] and np.isneginf(fs[2]) and t.id[2] == -1
