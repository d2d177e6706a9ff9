"""Pins for the oracle's stream / active-set functions (Eq. 3-5).

Each test checks the oracle against something other than itself: the worked
examples SPEC.md prints (tests/golden/spec_examples.json, each with its
citation), an independent characterisation of the window rule (last-occurrence
position instead of suffix slicing), invariants the paper states, and the
special cases the method reduces to.  CPU only.
"""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


def _gold():
    with open(GOLD) as f:
        return json.load(f)


# ---------------------------------------------------------------- golden (SPEC)
def test_golden_init():
    for case in _gold()["init"]:
        s, err = O.stream_init(case["prompt"], case["prefill"], case["vocab"])
        assert s.tolist() == case["stream"], case["cite"]
        assert err == 0
        for w, want in case.get("active", {}).items():
            ids, _ = O.active_set(s, case["vocab"], int(w))
            assert ids.tolist() == want, (case["cite"], w)


def test_golden_push():
    for case in _gold()["push"]:
        st = O.OracleStream(case["vocab"], case["w_max"]).init(case["prompt"])
        for draft, ver in case["updates"]:
            st.update(draft, ver)
        assert st.S.tolist() == case["stream"], case["cite"]
        assert st.active()[0].tolist() == case["active"], case["cite"]


def test_golden_suffix():
    for case in _gold()["suffix"]:
        ids, _ = O.active_set(np.asarray(case["stream"], np.int32), case["vocab"], case["w_max"])
        assert ids.tolist() == case["active"], case["cite"]


def test_golden_rules_differ_and_q2_counterexample():
    g = _gold()["rules"]
    a = g[0]
    assert O.active_set(a["stream"], a["vocab"], a["w_max"], O.RULE_WINDOW)[0].tolist() == a["active_R1"]
    assert O.active_set(a["stream"], a["vocab"], a["w_max"], O.RULE_UNIQUE_FIFO)[0].tolist() == a["active_R2"]
    b = g[1]
    for rule, key in ((O.RULE_WINDOW, "sizes_R1"), (O.RULE_UNIQUE_FIFO, "sizes_R2")):
        sizes = [len(O.active_set(b["stream"][:t], b["vocab"], b["w_max"], rule)[0])
                 for t in range(1, len(b["stream"]) + 1)]
        assert sizes == b[key], (b["cite"], key)


def test_golden_empty_prompt():
    case = _gold()["errors"][0]
    with pytest.raises(O.EmptyPrompt):
        O.stream_init(case["prompt"], None, 16)


# ------------------------------------------------- independent characterisation
def _r1_by_last_occurrence(S, W):
    """g in I  <=>  the most recent occurrence of g is among the last W stream
    positions ("tokens whose most recent occurrence falls outside the window are
    discarded")."""
    last = {}
    for p, g in enumerate(S):
        last[g] = p
    return sorted(g for g, p in last.items() if p >= len(S) - W)


def test_r1_exhaustive_tiny_streams():
    n = 0
    for V in (3, 4):
        for L in range(0, 7):
            for S in itertools.product(range(V), repeat=L):
                for W in (1, 2, 3, 4):
                    ids, bm = O.active_set(np.asarray(S, np.int32), V, W, O.RULE_WINDOW)
                    want = _r1_by_last_occurrence(S, W)
                    assert ids.tolist() == want, (S, W)
                    bits = [g for g in range(V) if (int(bm[g // 32]) >> (g % 32)) & 1]
                    assert bits == want
                    n += 1
    assert n > 20000


def test_r2_invariants_tiny_streams():
    """R2: |Q| = min(#pushes, W) is non-decreasing along the stream; Q holds the
    most recent W *distinct-at-push-time* entrants; W >= #distinct => Q = set(S)."""
    for V in (3, 4):
        for L in range(1, 7):
            for S in itertools.product(range(V), repeat=L):
                for W in (1, 2, 3):
                    prev = 0
                    for t in range(1, L + 1):
                        ids, _ = O.active_set(np.asarray(S[:t], np.int32), V, W, O.RULE_UNIQUE_FIFO)
                        assert len(ids) >= prev
                        assert len(ids) <= W
                        assert set(ids.tolist()) <= set(S[:t])
                        assert S[t - 1] in ids.tolist()  # the newest element is always a member
                        prev = len(ids)
                    if W >= len(set(S)):
                        assert ids.tolist() == sorted(set(S))


def test_stream_dedup_matches_order_preserving_dedup():
    """tuple(set) = first-occurrence order (Q3); compared with dict.fromkeys."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        V = int(rng.integers(2, 40))
        d = rng.integers(-2, V + 2, size=int(rng.integers(0, 70))).astype(np.int32)
        v = rng.integers(-2, V + 2, size=int(rng.integers(0, 5))).astype(np.int32)
        seg, err = O.stream_update(d, v, V)
        ok = lambda x: [int(t) for t in x if 0 <= t < V]
        want = list(dict.fromkeys(ok(d))) + list(dict.fromkeys(ok(v)))
        assert seg.tolist() == want
        assert err == int(any(not (0 <= t < V) for t in np.concatenate([d, v])))
        L = int(rng.integers(1, 20))
        prompt = rng.integers(0, V, size=L).astype(np.int32)
        pre = rng.integers(0, V, size=(L, 3)).astype(np.int32)
        s0, _ = O.stream_init(prompt, pre, V)
        assert s0.tolist() == prompt.tolist() + list(dict.fromkeys(pre.reshape(-1).tolist()))


def test_invariants_random_streams():
    """|I| <= W; I_{t+1} subset of I_t U batch; reads idempotent;
    W >= |S| => I = set(S) (seen-token special case); R1 monotone while |S| <= W."""
    rng = np.random.default_rng(11)
    for trial in range(300):
        V = int(rng.integers(4, 64))
        W = int(rng.choice([1, 4, 16, 64]))
        for rule in (O.RULE_WINDOW, O.RULE_UNIQUE_FIFO):
            st = O.OracleStream(V, W, rule).init(rng.integers(0, V, size=int(rng.integers(1, 30))))
            prev = set(st.active()[0].tolist())
            for _ in range(int(rng.integers(1, 12))):
                d = rng.integers(0, V, size=int(rng.integers(0, 9)))
                v = rng.integers(0, V, size=int(rng.integers(0, 4)))
                before_len = len(st.S)
                st.update(d, v)
                cur = st.active()[0].tolist()
                assert cur == st.active()[0].tolist()  # idempotent read
                assert len(cur) <= W
                assert set(cur) <= prev | set(d.tolist()) | set(v.tolist())
                if rule == O.RULE_WINDOW and len(st.S) <= W:
                    assert set(cur) >= prev and cur == sorted(set(st.S.tolist()))
                if rule == O.RULE_UNIQUE_FIFO:
                    assert len(cur) >= len(prev)
                prev = set(cur)
                assert before_len <= len(st.S)


def test_ring_reconstructs_the_window():
    """Reading the R1 ring from slot total%W onward gives Suffix(S, W) in order."""
    rng = np.random.default_rng(2)
    for _ in range(300):
        V = int(rng.integers(2, 50))
        W = int(rng.integers(1, 20))
        S = rng.integers(0, V, size=int(rng.integers(0, 60))).astype(np.int32)
        r, total = O.ring(S, V, W, O.RULE_WINDOW)
        assert total == len(S)
        if len(S) >= W:
            got = [int(r[(total + i) % W]) for i in range(W)]
            assert got == S[-W:].tolist()
        else:
            assert r[: len(S)].tolist() == S.tolist() and (r[len(S):] == -1).all()


def test_r2_ring_holds_queue():
    rng = np.random.default_rng(3)
    for _ in range(300):
        V = int(rng.integers(2, 30))
        W = int(rng.integers(1, 10))
        S = rng.integers(0, V, size=int(rng.integers(0, 40))).astype(np.int32)
        r, pushes = O.ring(S, V, W, O.RULE_UNIQUE_FIFO)
        ids, _ = O.active_set(S, V, W, O.RULE_UNIQUE_FIFO)
        live = [int(x) for x in r if x >= 0]
        assert sorted(live) == ids.tolist()
        assert pushes >= len(ids) and len(ids) == min(pushes, W)


def test_shards_partition_active_set():
    """Vocab-parallel shards (g % G == rank) partition I exactly."""
    rng = np.random.default_rng(4)
    for _ in range(100):
        V = int(rng.integers(8, 300))
        W = int(rng.integers(1, 100))
        S = rng.integers(0, V, size=int(rng.integers(1, 400))).astype(np.int32)
        full, _ = O.active_set(S, V, W)
        for G in (2, 3, 8):
            parts = []
            for r in range(G):
                ids, bm = O.active_set(S, V, W, O.RULE_WINDOW, r, G)
                assert all(int(g) % G == r for g in ids)
                local = [l for l in range(len(bm) * 32) if (int(bm[l // 32]) >> (l % 32)) & 1]
                assert local == [int(g) // G for g in ids]
                parts.extend(ids.tolist())
            assert sorted(parts) == full.tolist()


def test_invalid_ids_dropped_and_flagged():
    s, err = O.stream_init([3, 99, -1, 4], [[5, 77], [5, 6], [1, 2], [0, 0]], 10)
    assert err == 1 and s.tolist() == [3, 4, 5, 6, 1, 2, 0]


def test_init_with_k_pre_1():
    """Eq. 3 with K_pre = 1: S0 = prompt (+) tuple(first-ranked prefill
    candidate of every position), deduplicated within the union only."""
    s, err = O.stream_init([10, 11], [[12], [10]], 100)
    assert err == 0 and list(s) == [10, 11, 12, 10]
    ids4, _ = O.active_set(s, 100, 4)
    ids2, _ = O.active_set(s, 100, 2)
    assert list(ids4) == [10, 11, 12] and list(ids2) == [10, 12]
    # a repeated candidate inside the union is kept once, its first occurrence
    s, _ = O.stream_init([5], [[7]], 100)
    assert list(s) == [5, 7]
    s, _ = O.stream_init([5, 6, 8], [[7], [7], [9]], 100)
    assert list(s) == [5, 6, 8, 7, 9]
