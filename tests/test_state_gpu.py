"""GPU-resident state (a1/a2) vs the oracle, bit-exact: ids, n_active, bitmap,
ring, total (criterion 2 of S:636).  Calls through the C ABI."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from synthetic import inputs as SI

pytestmark = pytest.mark.gpu


def _t(a):
    return torch.as_tensor(np.asarray(a, np.int32), dtype=torch.int32, device="cuda").contiguous()


def _compare(st, seq, ref: O.OracleStream, shard_rank=0, n_shards=1, what=""):
    got = st.read(seq)
    ids, bm = ref.active(shard_rank, n_shards)
    assert got["n_active"] == len(ids), f"{what}: n_active {got['n_active']} vs {len(ids)}"
    assert np.array_equal(got["ids"], ids), what
    assert np.array_equal(got["bitmap"], bm), what
    ring, total = ref.ring()
    assert got["total"] == total, f"{what}: total {got['total']} vs {total}"
    assert np.array_equal(got["ring"], ring), what
    return got


@pytest.mark.parametrize("rule", ["window", "unique_fifo"])
def test_random_push_sequences(cuda_ok, rule):
    """Criterion 2: random streams, V <= 256, W_max in {1, 4, 16, 64}."""
    from paper_2605_26444_b200 import ActiveVocab
    rng = np.random.default_rng(17)
    orule = O.RULE_WINDOW if rule == "window" else O.RULE_UNIQUE_FIFO
    for trial in range(60):
        V = int(rng.integers(2, 257))
        W = int(rng.choice([1, 4, 16, 64]))
        st = ActiveVocab(V, W, rule=rule)
        ref = O.OracleStream(V, W, orule)
        prompt = rng.integers(0, V, size=int(rng.integers(1, 80)))
        pre = rng.integers(0, V, size=(len(prompt), int(rng.integers(0, 4))))
        st.init(0, _t(prompt), _t(pre) if pre.shape[1] else None)
        ref.init(prompt, pre if pre.shape[1] else None)
        _compare(st, 0, ref, what=f"trial {trial} init")
        for step in range(int(rng.integers(1, 25))):
            d = rng.integers(0, V, size=int(rng.integers(0, 70)))
            v = rng.integers(0, V, size=int(rng.integers(0, 4)))
            st.update(0, _t(d) if d.size else None, _t(v) if v.size else None)
            ref.update(d, v)
            _compare(st, 0, ref, what=f"trial {trial} step {step}")
        assert st.check() == 0


def test_spec_examples(cuda_ok):
    from paper_2605_26444_b200 import ActiveVocab
    st = ActiveVocab(32, 3)
    st.init(0, _t([10, 11]), _t([[11, 12], [10, 13]]))
    assert st.read(0)["ids"].tolist() == [10, 12, 13]
    st = ActiveVocab(16, 3)
    st.init(0, _t([1, 2, 3]))
    st.update(0, _t([4]), _t([5]))
    assert st.read(0)["ids"].tolist() == [3, 4, 5]


def test_empty_prompt_and_bad_ids(cuda_ok):
    from paper_2605_26444_b200 import ActiveVocab
    from paper_2605_26444_b200._native import NanoSpecError, EEMPTY
    st = ActiveVocab(16, 8)
    with pytest.raises(NanoSpecError) as e:
        st.init(0, torch.zeros(0, dtype=torch.int32, device="cuda"))
    assert e.value.status == EEMPTY
    st.init(0, _t([1, 2, 99, -3, 4]))
    got = st.read(0)
    assert got["ids"].tolist() == [1, 2, 4] and got["err"] == 1
    assert st.check() == 4  # EDEVICE


def test_tiny_config(cuda_ok):
    """BJ configs[0]: V=1000, 200-token Zipf prompt + K_pre=3, 5 steps of 8 tree
    tokens + 3 verify; W in {3072, 16, 64, 256}."""
    from paper_2605_26444_b200 import ActiveVocab
    z = SI.Zipf(1000)
    prompt, pre = SI.prompt_and_prefill(z, 2, 200, 3)
    steps = SI.decode_steps(z, 5, 5, n_draft=8, k_ver=3)
    for W in (3072, 16, 64, 256):
        st = ActiveVocab(1000, W)
        ref = O.OracleStream(1000, W).init(prompt, pre)
        st.init(0, _t(prompt), _t(pre))
        _compare(st, 0, ref, what=f"W={W} init")
        for i, (d, v) in enumerate(steps):
            st.update(0, _t(d), _t(v))
            ref.update(d, v)
            _compare(st, 0, ref, what=f"W={W} step {i}")


def test_qwen_replay(cuda_ok):
    """BJ configs[2]: Qwen-2.5-7B vocab, 2k-token prompt + K_pre=3, 512 steps of
    60 tree tokens + 3 verify; every 16th step and the final state compared."""
    from paper_2605_26444_b200 import ActiveVocab
    V, W = 152064, 3072
    z = SI.Zipf(V)
    prompt, pre = SI.prompt_and_prefill(z, 1, 2048, 3)
    steps = SI.decode_steps(z, 7, 512)
    st = ActiveVocab(V, W)
    ref = O.OracleStream(V, W).init(prompt, pre)
    st.init(0, _t(prompt), _t(pre))
    _compare(st, 0, ref, what="init")
    for i, (d, v) in enumerate(steps):
        st.update(0, _t(d), _t(v))
        ref.update(d, v)
        if i % 16 == 15 or i == len(steps) - 1:
            got = _compare(st, 0, ref, what=f"step {i}")
    assert 1500 < got["n_active"] <= W


def test_batch_update_and_shards(cuda_ok):
    """update_batch over B sequences == per-sequence oracle; vocab-parallel shards
    (cyclic, g % G == rank) == the oracle's shard of I."""
    from paper_2605_26444_b200 import ActiveVocab
    V, W, B = 5000, 300, 7
    z = SI.Zipf(V)
    st = ActiveVocab(V, W, batch=B)
    refs = []
    for b in range(B):
        p, pre = SI.prompt_and_prefill(z, 100 + b, 150, 3)
        st.init(b, _t(p), _t(pre))
        refs.append(O.OracleStream(V, W).init(p, pre))
    for step in range(12):
        rng = np.random.default_rng(step)
        d = np.stack([z.draw(rng, 60) for _ in range(B)])
        v = np.stack([z.draw_distinct(rng, 3) for _ in range(B)])
        st.update_batch(_t(d), _t(v))
        for b in range(B):
            refs[b].update(d[b], v[b])
    for b in range(B):
        _compare(st, b, refs[b], what=f"seq {b}")
    G = 4
    shards = [ActiveVocab(V, W, shard_rank=r, n_shards=G) for r in range(G)]
    p, pre = SI.prompt_and_prefill(z, 9, 400, 3)
    ref = O.OracleStream(V, W).init(p, pre)
    for s in shards:
        s.init(0, _t(p), _t(pre))
    for step in range(20):
        d, v = SI.decode_steps(z, 50 + step, 1)[0]
        ref.update(d, v)
        for s in shards:
            s.update(0, _t(d), _t(v))
    for r, s in enumerate(shards):
        _compare(s, 0, ref, r, G, what=f"shard {r}")


def test_long_update_batch_longer_than_window(cuda_ok):
    """Q8: an update batch longer than W_max -- only its last W_max slots survive."""
    from paper_2605_26444_b200 import ActiveVocab
    V, W = 3000, 50
    rng = np.random.default_rng(1)
    st = ActiveVocab(V, W)
    ref = O.OracleStream(V, W)
    p = rng.integers(0, V, size=30)
    st.init(0, _t(p))
    ref.init(p)
    for _ in range(5):
        d = rng.integers(0, V, size=2000)
        v = rng.integers(0, V, size=3)
        st.update(0, _t(d), _t(v))
        ref.update(d, v)
        _compare(st, 0, ref)


def test_ext_only_and_ctx_only_ablations(cuda_ok):
    """T5 ablation sources: Ext-only = no init, the active set comes
    from C_draft / C_ver alone (updates on a freshly created state); Ctx-only =
    init, then no updates (the state is left as S0).  Both bit-exact vs the oracle."""
    from paper_2605_26444_b200 import ActiveVocab
    rng = np.random.default_rng(23)
    V, W = 5000, 256
    st = ActiveVocab(V, W)
    ref = O.OracleStream(V, W)
    for step in range(12):  # Ext-only
        d = rng.integers(0, V, 60)
        v = rng.integers(0, V, 3)
        st.update(0, _t(d), _t(v))
        ref.update(d, v)
        _compare(st, 0, ref, what=f"ext-only step {step}")
    st2 = ActiveVocab(V, W)  # Ctx-only
    prompt = rng.integers(0, V, 400)
    pre = rng.integers(0, V, (400, 3))
    st2.init(0, _t(prompt), _t(pre))
    ref2 = O.OracleStream(V, W).init(prompt, pre)
    _compare(st2, 0, ref2, what="ctx-only")
