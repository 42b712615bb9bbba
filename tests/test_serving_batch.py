"""same-instant arrivals classified with one batched lookup must leave every
request, queue and simulation outcome exactly as the reference's one-lookup-per-arrival path
(scheduler.py:70-90, engine.py:201-209).  CPU: the drop-in over the FakeRing; the GPU variant
runs the same checks on the device ring."""
import dataclasses
import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
pytestmark = pytest.mark.skipif(not (REF / "mixserve").is_dir() and not Path("/root/reference/pkg/src").is_dir(),
                                reason="reference package not available")


def _mixserve():
    for p in (str(REF), "/root/reference/pkg/src"):
        if Path(p).is_dir() and p not in sys.path:
            sys.path.append(p)
    import mixserve.cache as mc
    import mixserve.config as mconfig
    import mixserve.engine as me
    import mixserve.scheduler as ms
    import mixserve.workload as mw

    return mc, mconfig, me, ms, mw


def _cache_cls(mc, gpu):
    from paper_2503_11972_b200 import SemanticCache, dropin

    base = SemanticCache
    if not gpu:
        from tests.fake_ring import FakeRing

        base = type("FakeRingCache", (SemanticCache,), {"_ring_factory": staticmethod(FakeRing)})
    return dropin.dropin_class(mc, base)


def _bursty_trace(mw, dim, n=240, seed=5):
    """Arrivals in bursts of 1-9 requests sharing one timestamp, clustered queries."""
    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((6, dim))
    out, t, i = [], 0.0, 0
    while i < n:
        t += float(rng.exponential(4000.0))
        for _ in range(int(rng.integers(1, 10))):
            v = centers[rng.integers(0, 6)] + 0.6 * rng.standard_normal(dim)
            out.append(mw.TraceRecord(f"r{i}", round(t, 3), v / np.linalg.norm(v)))
            i += 1
    return out[:n]


def run_classify_batch_matches_sequential(gpu=False):
    mc, mconfig, me, ms, mw = _mixserve()
    from paper_2503_11972_b200.serving import classify_batch

    Cache = _cache_cls(mc, gpu)
    rng = np.random.default_rng(3)
    d = 64
    caches = [Cache(capacity=300, dim=d), Cache(capacity=300, dim=d)]
    for c in caches:
        r2 = np.random.default_rng(4)
        for i in range(300):
            v = r2.standard_normal(d)
            c.insert(mc.CacheEntry(f"e{i}", v / np.linalg.norm(v), "large", i, float(i)))
    table = mc.ThresholdTable([(5, 0.5), (10, 0.6), (20, 0.8), (30, 0.9)])
    base = caches[0].entries()
    Q = [base[int(j)].embedding + 0.05 * rng.standard_normal(d) for j in rng.integers(0, 300, 40)]
    Q += [rng.standard_normal(d) for _ in range(10)]
    mk = lambda: [ms.Request(f"q{i}", 500.0, q / np.linalg.norm(q)) for i, q in enumerate(Q)]  # noqa: E731
    qa, qb = ms.QueuePair(), ms.QueuePair()
    seq = [ms.classify(r, caches[0], table, qa) for r in mk()]
    bat = classify_batch(mk(), caches[1], table, qb)
    strip = lambda r: {k: (v.tolist() if isinstance(v, np.ndarray) else v) for k, v in dataclasses.asdict(r).items()}  # noqa: E731
    assert [strip(r) for r in seq] == [strip(r) for r in bat]
    assert [r.id for r in qa.hit] == [r.id for r in qb.hit] and [r.id for r in qa.miss] == [r.id for r in qb.miss]
    assert qa.hit and qa.miss
    for c in caches:
        c.close()


def run_batched_arrivals_simulation_identical(gpu=False):
    mc, mconfig, me, ms, mw = _mixserve()
    from paper_2503_11972_b200.serving import install_batched_arrivals

    Cache = _cache_cls(mc, gpu)
    old = mc.SemanticCache
    mc.SemanticCache = mconfig.SemanticCache = Cache
    try:
        reports = []
        for batched in (False, True):
            cfg = mconfig.load_sim_config(_cfg_path("modm-cache-all.cfg"))
            cfg = dataclasses.replace(cfg, cache_dim=64, workload=dataclasses.replace(cfg.workload, dim=64))
            trace = _bursty_trace(mw, 64)
            sim = me.Simulation(cfg, trace)
            stats = install_batched_arrivals(sim, me) if batched else None
            res = sim.run()
            reports.append((json.dumps(dataclasses.asdict(res.report), sort_keys=True, default=str),
                            json.dumps(res.audit, sort_keys=True, default=str)))
            if batched:
                assert stats["batched_lookups"] > 100, stats  # most requests arrived in bursts
            sim.cache.close()
        assert reports[0] == reports[1]
    finally:
        mc.SemanticCache = mconfig.SemanticCache = old


def _cfg_path(name):
    for base in (REF / "configs", Path("/root/reference/pkg/configs")):
        if (base / name).exists():
            return base / name
    pytest.skip("reference configs not staged")


def test_classify_batch_matches_sequential_classify():
    run_classify_batch_matches_sequential(gpu=False)


def test_batched_arrivals_leave_the_simulation_unchanged():
    run_batched_arrivals_simulation_identical(gpu=False)


@pytest.mark.gpu
def test_classify_batch_on_gpu():
    run_classify_batch_matches_sequential(gpu=True)
    run_batched_arrivals_simulation_identical(gpu=True)
