"""Multi-process (gloo, world_size 2 and 3) tests of the sharded host path on CPU.

Every rank runs ShardedSemanticCache over a FakeShardRing (numpy float64
scan) and must return exactly the single-cache oracle's answers, through
capacity churn, age eviction and the insertion policy; the record exchange
is a real torch.distributed all-gather.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle.retrieval import OracleCache, OracleEntry, OracleTable
        from paper_2503_11972_b200 import CacheEntry, ThresholdTable
        from paper_2503_11972_b200.sharded import ShardedSemanticCache
        from tests.fake_shard_ring import FakeShardRing

        rng = np.random.default_rng(123)  # same stream on every rank (SPMD)
        d, cap = 24, 37
        table, ot = ThresholdTable.default(), OracleTable()
        centers = rng.standard_normal((5, d))
        # bulk preload of a capacity-only cache, then churn, against the oracle
        sb = ShardedSemanticCache(cap, d, policy="large", ring_factory=FakeShardRing)
        ob = OracleCache(cap, d, policy="large")
        pre = []
        for i in range(90):
            v = centers[i % 5] + 0.7 * rng.standard_normal(d)
            pre.append(CacheEntry(f"b{i}", v / np.linalg.norm(v), "small" if i % 7 == 0 else "large", i, float(i)))
        for chunk in (pre[:30], pre[30:]):  # the second chunk evicts part of the first
            evb = sb.bulk_load(chunk)
            evo = [x for e in chunk for x in ob.insert(OracleEntry(e.id, e.embedding, e.producer, e.seq, e.inserted_at))]
            assert [x.id for x in evb] == [x.id for x in evo], rank
        Qb = centers[rng.integers(0, 5, 6)] + 0.7 * rng.standard_normal((6, d))
        Qb /= np.linalg.norm(Qb, axis=1, keepdims=True)
        for q, r in zip(Qb, sb.retrieve_batch(Qb, table)):
            e, sim, k = ob.retrieve_entry(q, ot)
            assert (r.entry.id if r.hit else None) == (e.id if e is not None else None), rank
            assert r.k == k and abs(r.similarity - sim) < 1e-12
        sc = ShardedSemanticCache(cap, d, policy="all", max_age_s=60.0, ring_factory=FakeShardRing)
        oc = OracleCache(cap, d, max_age_s=60.0)
        t = 0.0
        for i in range(400):
            t += float(rng.exponential(1.0)) + (80.0 if i in (150, 151, 300) else 0.0)
            v = centers[i % 5] + 0.7 * rng.standard_normal(d)
            v /= np.linalg.norm(v)
            prod = "large" if rng.random() < 0.8 else "small"
            ev1 = sc.insert(CacheEntry(f"e{i}", v, prod, i, t))
            ev2 = oc.insert(OracleEntry(f"e{i}", v, prod, i, t))
            assert [e.id for e in ev1] == [e.id for e in ev2], (rank, i)
            assert len(sc) == len(oc.meta)
            if i % 9 == 0:
                Q = centers[rng.integers(0, 5, 4)] + 0.7 * rng.standard_normal((4, d))
                Q /= np.linalg.norm(Q, axis=1, keepdims=True)
                got = sc.retrieve_batch(Q, table)
                for q, r in zip(Q, got):
                    e, sim, k = oc.retrieve_entry(q, ot)
                    assert (r.entry.id if r.hit else None) == (e.id if e is not None else None), (rank, i)
                    assert r.k == k
                    assert (r.similarity is None) == (sim is None)
                    if sim is not None:
                        assert abs(r.similarity - sim) < 1e-12
        # shard sizes add up to the live window
        sizes = [None] * world
        dist.all_gather_object(sizes, len(sc.ring))
        assert sum(sizes) == len(sc), (sizes, len(sc))
        # degraded records (a failed certificate on some shard) went through the second round:
        # every rank rescanned and re-gathered together, and the answers above stayed exact
        rescans = [None] * world
        dist.all_gather_object(rescans, getattr(sc.ring, "rescans", 0))
        assert sum(rescans) > 0, rescans
        # pipelined lookups over the process group: futures complete in the same order on every
        # rank, so the rescan round's all-gather stays SPMD
        sp = ShardedSemanticCache(cap, d, max_age_s=60.0, ring_factory=FakeShardRing)
        from tests.test_sharded_gloo import _pipelined_against_oracle

        assert _pipelined_against_oracle(sp, d, cap, steps=150) > 150
        dist.destroy_process_group()
    except BaseException as exc:  # pragma: no cover - reported to the parent
        import traceback

        errq.put(f"rank {rank}: {exc!r}\n{traceback.format_exc()}")
        raise


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_cache_matches_oracle_over_gloo(world):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    errors = []
    while not errq.empty():
        errors.append(errq.get())
    assert not errors, "\n".join(errors)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


def test_count_owned():
    from paper_2503_11972_b200.sharded import _count_owned

    for G in (1, 2, 3, 8):
        for g in range(G):
            for lo in range(0, 20):
                for n in range(0, 20):
                    want = sum(1 for p in range(lo, lo + n) if p % G == g)
                    assert _count_owned(lo, n, g, G) == want


def _churn_against_oracle(make_cache, d=24, cap=37, steps=400, seed=123, B=4, check_every=9):
    """Insert / evict / lookup churn (policy, age, capacity) vs the single-cache oracle."""
    from oracle.retrieval import OracleCache, OracleEntry, OracleTable
    from paper_2503_11972_b200 import CacheEntry, ThresholdTable

    rng = np.random.default_rng(seed)
    table, ot = ThresholdTable.default(), OracleTable()
    centers = rng.standard_normal((5, d))
    sc = make_cache(cap, d, "all", 60.0)
    oc = OracleCache(cap, d, max_age_s=60.0)
    t = 0.0
    n_checked = 0
    for i in range(steps):
        t += float(rng.exponential(1.0)) + (80.0 if i in (150, 151, 300) else 0.0)
        v = centers[i % 5] + 0.7 * rng.standard_normal(d)
        v /= np.linalg.norm(v)
        prod = "large" if rng.random() < 0.8 else "small"
        ev1 = sc.insert(CacheEntry(f"e{i}", v, prod, i, t))
        ev2 = oc.insert(OracleEntry(f"e{i}", v, prod, i, t))
        assert [e.id for e in ev1] == [e.id for e in ev2], i
        assert len(sc) == len(oc.meta) == sum(sc.shard_sizes())
        if i % check_every == 0:
            Q = centers[rng.integers(0, 5, B)] + 0.7 * rng.standard_normal((B, d))
            Q /= np.linalg.norm(Q, axis=1, keepdims=True)
            for q, r in zip(Q, sc.retrieve_batch(Q, table)):
                e, sim, k = oc.retrieve_entry(q, ot)
                assert (r.entry.id if r.hit else None) == (e.id if e is not None else None), i
                assert r.k == k and (r.similarity is None) == (sim is None)
                if sim is not None:
                    assert abs(r.similarity - sim) < 1e-12
                n_checked += 1
    sizes = sc.shard_sizes()
    assert max(sizes) - min(sizes) <= 1, sizes  # round-robin keeps the shards balanced
    sc.close()
    return n_checked


@pytest.mark.parametrize("G", [1, 2, 3, 8])
def test_local_shards_match_oracle_on_cpu(G):
    """local_shards mode (every shard in one process, records written into one buffer, no
    collective) over FakeShardRing: the host bookkeeping of the single-process sharded path."""
    from paper_2503_11972_b200.sharded import ShardedSemanticCache
    from tests.fake_shard_ring import FakeShardRing

    n = _churn_against_oracle(lambda cap, d, pol, age: ShardedSemanticCache(
        cap, d, policy=pol, max_age_s=age, ring_factory=FakeShardRing, local_shards=G))
    assert n > 100


def _pipelined_against_oracle(sc, d, cap, steps=300, seed=321):
    """retrieve_async / retrieve_batch_async submitted before the request's insert and read one
    request later (two pending), through capacity and age churn: every answer is the oracle's at
    its submit state, entries by id."""
    from oracle.retrieval import OracleCache, OracleEntry, OracleTable
    from paper_2503_11972_b200 import CacheEntry, ThresholdTable

    rng = np.random.default_rng(seed)
    table, ot = ThresholdTable.default(), OracleTable()
    centers = rng.standard_normal((5, d))
    oc = OracleCache(cap, d, max_age_s=60.0)
    t, prev, n_checked = 0.0, None, 0

    def check(res, want):
        nonlocal n_checked
        res = [res] if not isinstance(res, list) else res
        for r, (e, sim, k) in zip(res, want):
            assert (r.entry.id if r.hit else None) == (e.id if e is not None else None)
            assert r.k == k and (r.similarity is None) == (sim is None)
            if sim is not None:
                assert abs(r.similarity - sim) < 1e-12
            n_checked += 1

    for i in range(steps):
        t += float(rng.exponential(1.0)) + (80.0 if i in (120, 240) else 0.0)
        B = 1 if i % 3 else 3
        Q = centers[rng.integers(0, 5, B)] + 0.7 * rng.standard_normal((B, d))
        Q /= np.linalg.norm(Q, axis=1, keepdims=True)
        want = [oc.retrieve_entry(q, ot) for q in Q]
        fut = sc.retrieve_async(Q[0], table) if B == 1 else sc.retrieve_batch_async(Q, table)
        v = centers[i % 5] + 0.7 * rng.standard_normal(d)
        v /= np.linalg.norm(v)
        sc.insert(CacheEntry(f"e{i}", v, "large", i, t))
        oc.insert(OracleEntry(f"e{i}", v, "large", i, t))
        if prev is not None:
            check(prev[0].result(), prev[1])
        prev = (fut, want)
    check(prev[0].result(), prev[1])
    return n_checked


@pytest.mark.parametrize("G", [1, 3])
def test_local_shards_pipelined_lookups_on_cpu(G):
    """ShardedSemanticCache.retrieve_async / retrieve_batch_async over FakeShardRing (degraded
    records every third query: the rescan round runs at result time)."""
    from paper_2503_11972_b200.sharded import ShardedSemanticCache
    from tests.fake_shard_ring import FakeShardRing

    sc = ShardedSemanticCache(37, 24, max_age_s=60.0, ring_factory=FakeShardRing, local_shards=G)
    assert _pipelined_against_oracle(sc, 24, 37) > 300
    assert sum(getattr(r, "rescans", 0) for r in sc._rings.values()) > 0
