"""Bulk preload / snapshot import: SemanticCache.bulk_load and the chunked
import_jsonl must equal the reference's per-entry insert() replay (cache.py:206-235, 279-302) in
every observable — stored entries, evictions, next_seq, errors and their messages (CPU, fake ring)."""
import json

import numpy as np
import pytest

import paper_2503_11972_b200.cache as cache_mod
from paper_2503_11972_b200 import CacheEntry, EmbeddingError, SemanticCache, normalize
from tests.fake_ring import FakeRing


@pytest.fixture(autouse=True)
def fake_ring(monkeypatch):
    monkeypatch.setattr(cache_mod.SemanticCache, "_ring_factory", staticmethod(FakeRing))


def _entries(rng, n, d, seq0=0, small_every=0):
    out = []
    for i in range(n):
        prod = "small" if small_every and i % small_every == 0 else "large"
        out.append(CacheEntry(f"e{seq0 + i}", normalize(rng.standard_normal(d)), prod, seq0 + i, float(i)))
    return out


def _state(c):
    return [e.id for e in c.entries()], c.next_seq, [r.tolist() for r in c.ring.rows]


@pytest.mark.parametrize("policy", ["all", "large"])
@pytest.mark.parametrize("cap,n", [(50, 30), (50, 50), (50, 120), (7, 1000)])
def test_bulk_equals_sequential_inserts(policy, cap, n):
    rng = np.random.default_rng(cap * 1000 + n)
    d = 8
    pre = _entries(rng, 20, d)
    batch = _entries(rng, n, d, seq0=100, small_every=3)
    a, b = SemanticCache(cap, d, policy=policy), SemanticCache(cap, d, policy=policy)
    for e in pre:
        a.insert(e)
        b.insert(e)
    ev_seq = [x.id for e in batch for x in a.insert(e)]
    ev_bulk = [x.id for x in b.bulk_load(batch)]
    assert ev_bulk == ev_seq
    assert _state(a) == _state(b)


def test_bulk_stops_at_the_first_invalid_entry_like_insert():
    rng = np.random.default_rng(5)
    d = 6
    good = _entries(rng, 10, d)
    bad_norm = CacheEntry("bad", 2.0 * good[0].embedding, "large", 10, 0.0)
    rest = _entries(rng, 5, d, seq0=11)
    for bad, exc, msg in [(bad_norm, EmbeddingError, "not unit norm"),
                          (CacheEntry("shape", np.ones(d + 1) / np.sqrt(d + 1), "large", 10, 0.0), EmbeddingError,
                           "shape"),
                          (CacheEntry("prod", good[0].embedding, "medium", 10, 0.0), ValueError, "unknown producer"),
                          (CacheEntry("seq", good[0].embedding, "large", 3, 0.0), ValueError, "seq must increase")]:
        a, b = SemanticCache(40, d), SemanticCache(40, d)
        with pytest.raises(exc, match=msg) as e1:
            for e in good + [bad] + rest:
                a.insert(e)
        with pytest.raises(exc, match=msg) as e2:
            b.bulk_load(good + [bad] + rest)
        assert str(e1.value) == str(e2.value)
        assert _state(a) == _state(b)


def test_bulk_with_age_limit_matches_inserts():
    rng = np.random.default_rng(9)
    d = 4
    batch = _entries(rng, 60, d)
    batch = [CacheEntry(e.id, e.embedding, e.producer, e.seq, 10.0 * i) for i, e in enumerate(batch)]
    a, b = SemanticCache(100, d, max_age_s=95.0), SemanticCache(100, d, max_age_s=95.0)
    ev_seq = [x.id for e in batch for x in a.insert(e)]
    assert [x.id for x in b.bulk_load(batch)] == ev_seq
    assert _state(a) == _state(b)


def test_chunked_import_equals_per_line_replay(tmp_path):
    rng = np.random.default_rng(2)
    d = 5
    path = tmp_path / "snap.jsonl"
    ents = _entries(rng, 9000, d, small_every=4)
    with open(path, "w") as fh:
        for e in ents:
            fh.write(json.dumps({"id": e.id, "seq": e.seq, "inserted_at": e.inserted_at, "producer": e.producer,
                                 "embedding": e.embedding.tolist()}) + "\n")
    a = SemanticCache(5000, d, policy="large")
    ref_acc = 0
    for e in ents:  # the reference's loop (cache.py:279-302)
        before = a.next_seq
        a.insert(e)
        ref_acc += a.next_seq != before
    b = SemanticCache(5000, d, policy="large")
    assert b.import_jsonl(path) == ref_acc
    assert _state(a) == _state(b)
    with open(path, "a") as fh:
        fh.write("{not json\n")
    c = SemanticCache(5000, d, policy="large")
    with pytest.raises(ValueError, match=r"snap.jsonl:9001: bad snapshot record"):
        c.import_jsonl(path)
    assert _state(c) == _state(a)  # every record before the bad line was stored


def test_async_lookup_resolves_against_its_submit_state():
    """retrieve_async + insert (capacity evictions) + result() == retrieve() before the insert."""
    rng = np.random.default_rng(17)
    d, cap = 8, 40
    a, b = SemanticCache(cap, d), SemanticCache(cap, d)
    from paper_2503_11972_b200 import ThresholdTable

    table = ThresholdTable.default()
    ents = _entries(rng, 2000, d)
    for e in ents[:cap]:
        a.insert(e)
        b.insert(e)
    for i, e in enumerate(ents[cap:]):
        q = normalize(ents[cap + i - 3].embedding + 0.3 * rng.standard_normal(d))
        want = a.retrieve(q, table)
        a.insert(e)
        pend = b.retrieve_async(q, table)
        b.insert(e)  # evicts the oldest entry while the lookup is pending
        got = pend.result()
        assert got == want, i
        assert (got.entry is want.entry) or got.entry is None
    assert _state(a) == _state(b)


def test_serving_decisions_follow_the_reference_rules():
    """route = hit queue (scheduler.py:80-89), steps = T - k (engine.py:38-45),
    sigma = noise_reentry_level(k, schedule) (cache.py:305-334), per query, from one batched lookup."""
    from paper_2503_11972_b200 import ThresholdTable, linear_sigma_schedule, noise_reentry_level

    rng = np.random.default_rng(23)
    d = 256
    c = SemanticCache(200, d)
    ents = _entries(rng, 150, d)
    c.bulk_load(ents)
    table = ThresholdTable.default(total_steps=50)
    sched = linear_sigma_schedule(50)
    Q = np.stack([normalize(ents[i].embedding + s * rng.standard_normal(d) / np.sqrt(d))
                  for i, s in zip(rng.integers(0, 150, 64), np.linspace(0.05, 8.0, 64))]
                 + [normalize(rng.standard_normal(d)) for _ in range(16)])
    dec = c.serving_decisions(Q, table, sched)
    for q, row in zip(Q, dec):
        r = c.retrieve(q, table)
        assert row["hit"] == r.hit and row["route"] == int(r.hit)
        assert row["similarity"] == r.similarity
        assert row["k"] == (r.k or 0) and row["steps"] == 50 - (r.k or 0)
        if r.hit:
            assert c.entries()[row["live"]] is r.entry
            assert row["sigma"] == noise_reentry_level(r.k, sched)
        else:
            assert row["live"] == -1 and np.isnan(row["sigma"])
    assert dec["hit"].any() and (~dec["hit"]).any()
    empty = SemanticCache(10, d).serving_decisions(Q[:3], table, sched)
    assert (empty["live"] == -1).all() and (empty["steps"] == 50).all() and not empty["hit"].any()


def test_fast_result_objects_equal_dataclass_ones():
    """retrieve_batch builds its RetrievalResult objects without the dataclass __init__;
    they must be indistinguishable from ones built the normal way (and stay frozen)."""
    import dataclasses

    import pytest

    from paper_2503_11972_b200.records import CacheEntry, RetrievalResult, make_result

    e = CacheEntry("x", np.ones(4) / 2.0, "large", 0, 0.0)
    for args in ((e, 0.75, 10), (None, 0.125, None)):
        a, b = make_result(*args), RetrievalResult(*args)
        assert type(a) is RetrievalResult and a == b and repr(a) == repr(b) and a.hit == b.hit
        assert (a.entry, a.similarity, a.k) == (b.entry, b.similarity, b.k)
        with pytest.raises(dataclasses.FrozenInstanceError):
            a.k = 1


def test_async_batches_resolve_against_their_submit_state():
    """retrieve_batch_async pipelined one deep (batch i+1 submitted before batch i is read), with
    inserts and capacity evictions between: every RetrievalBatch equals retrieve_batch() at its
    submit time, entries by identity; a dropped future is completed by the next lookup."""
    from paper_2503_11972_b200 import ThresholdTable

    rng = np.random.default_rng(29)
    d, cap = 8, 40
    a, b = SemanticCache(cap, d), SemanticCache(cap, d)
    table = ThresholdTable.default()
    ents = _entries(rng, 400, d)
    for e in ents[:cap]:
        a.insert(e)
        b.insert(e)
    prev = None
    for i, e in enumerate(ents[cap:]):
        Q = np.stack([normalize(ents[cap + i - j].embedding + 0.3 * rng.standard_normal(d)) for j in (1, 5, 9)])
        want = a.retrieve_batch(Q, table)
        a.insert(e)
        pend = b.retrieve_batch_async(Q, table)
        b.insert(e)
        if prev is not None:
            got, exp = prev[0].result(), prev[1]
            assert list(got) == list(exp), i
            assert all(x.entry is y.entry for x, y in zip(got, exp))
            assert np.array_equal(got.similarity, exp.similarity) and np.array_equal(got.k, exp.k)
        prev = (pend, want)
        if i % 50 == 49:  # dropped future: the next lookup completes it
            b.retrieve_batch_async(Q, table)
            want2 = a.retrieve_batch(Q, table)
            assert list(b.retrieve_batch(Q, table)) == list(want2)
            prev = None
    assert _state(a) == _state(b)
