"""Host-side logic of the drop-in SemanticCache (CPU; device ring replaced by a test fake).

Mirrors the reference's own unit tests (pkg/tests/test_cache.py:31-309) for
everything that is decided on the host: validation order and exception
types, FIFO / policy / age bookkeeping, snapshot round trips, result mapping.
"""
import numpy as np
import pytest

import paper_2503_11972_b200.cache as cache_mod
from paper_2503_11972_b200 import (
    CacheEntry,
    EmbeddingError,
    RetrievalResult,
    SemanticCache,
    ThresholdTable,
    cosine,
    linear_sigma_schedule,
    noise_reentry_level,
    normalize,
    validate_sigma_schedule,
)
from tests.fake_ring import FakeRing
from tests.golden_replay import SCENARIOS, expected, load, replay


@pytest.fixture(autouse=True)
def fake_ring(monkeypatch):
    monkeypatch.setattr(cache_mod.SemanticCache, "_ring_factory", staticmethod(FakeRing))


def unit(rng, d):
    return normalize(rng.standard_normal(d))


def entry(seq, emb, producer="large", t=0.0, eid=None):
    return CacheEntry(eid or f"e{seq}", emb, producer, seq, t)


class TestValidation:
    def test_constructor_errors(self):
        with pytest.raises(ValueError):
            SemanticCache(capacity=0)
        with pytest.raises(ValueError):
            SemanticCache(capacity=4, policy="bogus")
        with pytest.raises(ValueError):
            SemanticCache(capacity=4, max_age_s=0)

    def test_policy_drop_precedes_validation(self):
        c = SemanticCache(capacity=4, dim=8, policy="large")
        # a small-producer entry with a bad shape is silently dropped, not rejected (cache.py:211-212)
        assert c.insert(CacheEntry("x", np.ones(3), "small", 0, 0.0)) == []

    def test_unknown_producer(self):
        with pytest.raises(ValueError):
            SemanticCache(capacity=4, dim=8).insert(entry(0, unit(np.random.default_rng(0), 8), producer="mid"))

    def test_shape_norm_seq(self):
        rng = np.random.default_rng(1)
        c = SemanticCache(capacity=4, dim=8)
        with pytest.raises(EmbeddingError):
            c.insert(entry(0, unit(rng, 7)))
        with pytest.raises(EmbeddingError):
            c.insert(CacheEntry("x", np.full(8, 0.5), "large", 0, 0.0))
        c.insert(entry(5, unit(rng, 8)))
        with pytest.raises(ValueError):
            c.insert(entry(5, unit(rng, 8)))

    def test_query_shape(self):
        c = SemanticCache(capacity=4, dim=8)
        with pytest.raises(EmbeddingError):
            c.retrieve(normalize([1.0, 0.0]), ThresholdTable.default())

    def test_empty_cache_never_touches_device(self):
        c = SemanticCache(capacity=4, dim=8)
        assert c.retrieve(unit(np.random.default_rng(2), 8), ThresholdTable.default()) == RetrievalResult(None, None, None)
        assert c._ring is None


class TestBookkeeping:
    def test_fifo_eviction_mirrors_ring(self):
        rng = np.random.default_rng(3)
        c = SemanticCache(capacity=2, dim=8)
        es = [entry(i, unit(rng, 8), t=float(i), eid=n) for i, n in enumerate("abc")]
        assert c.insert(es[0]) == [] and c.insert(es[1]) == []
        assert [e.id for e in c.insert(es[2])] == ["a"]
        assert [e.id for e in c.entries()] == ["b", "c"]
        assert len(c.ring) == len(c) == 2

    def test_age_eviction_on_next_insert(self):
        rng = np.random.default_rng(4)
        c = SemanticCache(capacity=10, dim=8, max_age_s=4 * 3600.0)
        c.insert(entry(0, unit(rng, 8), t=0.0, eid="stale"))
        assert len(c) == 1
        assert [e.id for e in c.insert(entry(1, unit(rng, 8), t=5 * 3600.0, eid="fresh"))] == ["stale"]
        assert len(c.ring) == 1

    def test_policy_is_mutable(self):
        c = SemanticCache(capacity=4, dim=8)
        c.policy = "disabled"
        assert not c.admits("large")

    def test_retained_set_is_most_recent_eligible(self):
        rng = np.random.default_rng(5)
        c = SemanticCache(capacity=5, dim=8, policy="large")
        eligible = []
        for i in range(40):
            producer = "large" if rng.random() < 0.6 else "small"
            c.insert(entry(i, unit(rng, 8), producer=producer, t=float(i)))
            if producer == "large":
                eligible.append(f"e{i}")
        assert [e.id for e in c.entries()] == eligible[-5:]
        assert len(c.ring) == 5


def _retrieve(cache, q, table):
    r = cache.retrieve(q, table)
    live = None
    if r.hit:
        live = [e.seq for e in cache.entries()].index(r.entry.seq)
    return (r.entry.seq if r.hit else None), live, r.similarity, r.k


@pytest.mark.parametrize("name", SCENARIOS)
def test_host_logic_replays_golden(name):
    g = load(name)
    got = replay(g, lambda cap, dim, pol, age: SemanticCache(cap, dim, pol, age), CacheEntry,
                 lambda pairs, T: ThresholdTable(pairs, T), _retrieve)
    want = expected(g)
    for a, b in zip(got, want):
        assert (a[0], a[1], a[3]) == (b[0], b[1], b[3])
        assert (a[2] is None) == (b[2] is None)
        if a[2] is not None:
            assert abs(a[2] - b[2]) <= 1e-12


def test_snapshot_round_trip(tmp_path):
    rng = np.random.default_rng(10)
    c = SemanticCache(capacity=20, dim=8)
    for i in range(12):
        c.insert(entry(i, unit(rng, 8), producer=("small" if i % 4 else "large"), t=i * 2.5))
    p1, p2 = tmp_path / "a.jsonl", tmp_path / "b.jsonl"
    c.export_jsonl(p1)
    c2 = SemanticCache(capacity=20, dim=8)
    assert c2.import_jsonl(p1) == 12
    c2.export_jsonl(p2)
    assert p1.read_bytes() == p2.read_bytes()
    bad = tmp_path / "bad.jsonl"
    bad.write_text('{"id": "a", "seq": 0}\n', encoding="utf-8")
    with pytest.raises(ValueError, match="bad.jsonl:1"):
        SemanticCache(capacity=4, dim=8).import_jsonl(bad)


class TestPureHelpers:
    def test_table(self):
        t = ThresholdTable.default()
        assert t.step_choices == (5, 10, 15, 20, 25, 30) and t.tau == 0.25
        for s, k in [(0.305, 30), (0.265, 10), (1.0, 30), (0.25, 5), (0.2499999, None), (-1.0, None)]:
            assert t.select_k(s) == k
        for bad in ([(10, 0.3), (5, 0.2)], [(5, 0.3), (10, 0.2)], [], [(5, 1.5)]):
            with pytest.raises(ValueError):
                ThresholdTable(bad)
        with pytest.raises(ValueError):
            ThresholdTable([(5, 0.2), (50, 0.3)], total_steps=50)

    def test_vectors(self):
        assert np.allclose(normalize([3.0, 4.0]), [0.6, 0.8])
        for bad in ([0.0, 0.0], [1.0, np.nan], [np.inf, 0.0]):
            with pytest.raises(EmbeddingError):
                normalize(bad)
        assert cosine(normalize([3.0, 4.0]), normalize([4.0, 3.0])) == pytest.approx(0.96)
        with pytest.raises(EmbeddingError):
            cosine(normalize([1.0, 0.0]), normalize([1.0, 0.0, 0.0]))

    def test_schedule(self):
        s = linear_sigma_schedule(50)
        validate_sigma_schedule(s)
        assert noise_reentry_level(0, s) == 1.0 and noise_reentry_level(50, s) == 0.0
        with pytest.raises(ValueError):
            noise_reentry_level(51, s)
        with pytest.raises(ValueError):
            validate_sigma_schedule(np.array([1.0, 0.2, 0.5, 0.0]))


class TestAsyncLifecycle:
    """a dropped retrieve_async future must not wedge the cache or its FIFO pin."""

    def test_dropped_future_is_completed_by_the_next_lookup(self):
        rng = np.random.default_rng(3)
        c = SemanticCache(capacity=4, dim=8)
        for i in range(4):
            c.insert(entry(i, unit(rng, 8)))
        q = unit(rng, 8)
        fut = c.retrieve_async(q, ThresholdTable.default())
        want = c._ring.retrieve1(q)  # the answer for the state at submit time
        del fut  # never .result()-ed
        for i in range(4, 2100):  # churn past the compaction threshold: the pin must be released
            c.insert(entry(i, unit(rng, 8)))
        r = c.retrieve(q, ThresholdTable.default())  # completes the dropped lookup first
        assert not c._pending and c._store._pins == 0
        c.insert(entry(2100, unit(rng, 8)))
        assert len(c._store._items) < 100  # compaction runs again once unpinned
        assert r.similarity is not None and want is not None

    def test_result_is_kept_after_a_later_lookup_completed_it(self):
        rng = np.random.default_rng(4)
        c = SemanticCache(capacity=16, dim=8)
        for i in range(16):
            c.insert(entry(i, unit(rng, 8)))
        q = c.entries()[5].embedding
        fut = c.retrieve_async(q, ThresholdTable.default())
        c.insert(entry(16, unit(rng, 8)))  # evicts e0 while the lookup is pending
        c.retrieve_batch(np.stack([q, q]), ThresholdTable.default())  # settles the pending lookup
        r = fut.result()
        assert r.hit and r.entry.id == "e5" and r.k == 30

    def test_out_of_window_device_index_fails_loudly(self):
        from paper_2503_11972_b200 import _native

        class BadRing(FakeRing):
            def retrieve1(self, q):
                live, sim, k, flags = super().retrieve1(q)
                return -1, sim, k, flags | _native.MC_FLAG_HIT

        c = SemanticCache(capacity=4, dim=8)
        c._ring = BadRing(4, 8)
        rng = np.random.default_rng(5)
        for i in range(3):
            c.insert(entry(i, unit(rng, 8)))
        with pytest.raises(_native.NativeError, match="outside the window"):
            c.retrieve(unit(rng, 8), ThresholdTable.default())


def test_threshold_table_nan_message_matches_the_reference():
    """with a NaN tau the reference's `any(b <= a)` passes and the range check
    raises; the messages must match (cache.py:84-93)."""
    with pytest.raises(ValueError, match="thresholds must lie in"):
        ThresholdTable([(5, 0.25), (10, float("nan"))])
    with pytest.raises(ValueError, match="thresholds must lie in"):
        ThresholdTable([(5, float("nan")), (10, 0.3), (15, 0.4)])
    with pytest.raises(ValueError, match="strictly increasing"):
        ThresholdTable([(5, 0.3), (10, 0.3)])


class TestPipelinedAndBatchResults:
    def test_pending_lookups_answer_for_their_own_submit_state(self):
        """Up to three retrieve_async lookups in flight: each answers for the cache as it was when
        submitted; a fourth submit completes the oldest first."""
        rng = np.random.default_rng(11)
        c = SemanticCache(capacity=8, dim=8)
        for i in range(8):
            c.insert(entry(i, unit(rng, 8)))
        table = ThresholdTable.default()
        q0 = c.entries()[0].embedding  # e0: evicted by the next insert
        f0 = c.retrieve_async(q0, table)
        c.insert(entry(8, unit(rng, 8)))
        q1 = c.entries()[0].embedding  # e1: evicted by the next insert
        f1 = c.retrieve_async(q1, table)
        assert len(c._pending) == 2
        c.insert(entry(9, unit(rng, 8)))
        q2 = c.entries()[0].embedding  # e2: evicted by the next insert
        f2 = c.retrieve_async(q2, table)
        assert len(c._pending) == 3 and f0._cache is not None
        c.insert(entry(10, unit(rng, 8)))
        f3 = c.retrieve_async(c.entries()[-1].embedding, table)  # completes f0 first
        assert len(c._pending) == 3 and f0._cache is None
        assert f1.result().entry.id == "e1" and f0.result().entry.id == "e0" and f2.result().entry.id == "e2"
        assert f3.result().entry.id == "e10"
        assert not c._pending and c._store._pins == 0
        # beside a batch, two: a single submit with a batch pending completes down to one
        fb = c.retrieve_batch_async(np.stack([c.entries()[1].embedding, c.entries()[2].embedding]), table)
        fs = c.retrieve_async(c.entries()[3].embedding, table)
        fs2 = c.retrieve_async(c.entries()[4].embedding, table)  # completes the batch first
        assert fb._cache is None and len(c._pending) == 2
        assert [r.entry.id for r in fb.result()] == ["e4", "e5"] and fs.result().entry.id == "e6"
        assert fs2.result().entry.id == "e7"

    def test_a_new_table_settles_pending_lookups(self):
        rng = np.random.default_rng(12)
        c = SemanticCache(capacity=8, dim=8)
        for i in range(8):
            c.insert(entry(i, unit(rng, 8)))
        f = c.retrieve_async(c.entries()[3].embedding, ThresholdTable.default())
        other = ThresholdTable([(5, 0.2), (10, 0.9)], 50)
        r = c.retrieve(c.entries()[3].embedding, other)
        assert not c._pending and f.result().k == 30 and r.k == 10

    def test_retrieval_batch_is_the_list_of_answers(self):
        from paper_2503_11972_b200 import RetrievalBatch

        rng = np.random.default_rng(13)
        c = SemanticCache(capacity=32, dim=8)
        for i in range(32):
            c.insert(entry(i, unit(rng, 8)))
        table = ThresholdTable.default()
        Q = np.stack([c.entries()[5].embedding] + [unit(rng, 8) for _ in range(6)])
        got = c.retrieve_batch(Q, table)
        want = [c.retrieve(q, table) for q in Q]
        assert isinstance(got, RetrievalBatch) and len(got) == len(Q)
        assert got == want and list(got) == want and got[0] == want[0] and got[-1] == want[-1]
        assert got.hit.tolist() == [r.hit for r in want]
        assert np.allclose(got.similarity, [r.similarity for r in want])
        fresh = c.retrieve_batch(Q, table)  # no item built yet
        for j in range(40):  # later inserts evict the hit entries: the batches keep their answers
            c.insert(entry(100 + j, unit(rng, 8)))
        assert fresh[0].entry.id == "e5" and fresh == want and got == want
        assert SemanticCache(capacity=4, dim=8).retrieve_batch(Q[:2], table) == [RetrievalResult(None, None, None)] * 2


def test_add_mints_ordinary_entries_for_every_policy():
    """add() builds entries without the dataclass __init__ (records._entry_factory): they must be
    ordinary instances (equality, hash, repr, frozen), for ours and a drop-in's entry class; the
    inlined admits() must agree with admits() for every policy and producer."""
    import dataclasses
    import types

    from paper_2503_11972_b200 import dropin

    rng = np.random.default_rng(3)
    e = unit(rng, 8)
    c = SemanticCache(capacity=4, dim=8)
    c.add("a", e, "large", 1.5)
    got = c.entries()[0]
    want = CacheEntry("a", e, "large", 0, 1.5)
    assert type(got) is CacheEntry and got == want and repr(got) == repr(want)
    with pytest.raises(dataclasses.FrozenInstanceError):
        got.seq = 3

    @dataclasses.dataclass(frozen=True)
    class OtherEntry:
        id: str
        embedding: np.ndarray
        producer: str
        seq: int
        inserted_at: float

    mod = types.SimpleNamespace(CacheEntry=OtherEntry, EmbeddingError=EmbeddingError,
                                RetrievalResult=RetrievalResult)
    d = dropin.dropin_class(mod)(capacity=4, dim=8)
    d.add("b", e, "small", 2.0)
    assert d.entries()[0] == OtherEntry("b", e, "small", 0, 2.0)

    for policy in ("all", "large", "disabled"):
        for producer in ("large", "small"):
            c = SemanticCache(capacity=4, dim=8, policy=policy)
            c.add("x", e, producer, 0.0)
            assert len(c) == int(c.admits(producer)), (policy, producer)
