"""Pin the CPU oracle against the reference's own outputs (golden op logs) and KATs."""
import numpy as np
import pytest

from oracle.retrieval import OracleCache, OracleEntry, OracleTable, scan_oracle
from tests.golden_replay import SCENARIOS, expected, load, replay


def _oracle_retrieve(cache, q, table):
    live, sim, k = cache.retrieve(q, table)
    seq = cache.meta[live].seq if live is not None else None
    return seq, live, sim, k


@pytest.mark.parametrize("name", SCENARIOS)
def test_oracle_matches_reference_golden(name):
    g = load(name)
    got = replay(
        g,
        lambda cap, dim, pol, age: OracleCache(cap, dim, pol, age),
        OracleEntry,
        OracleTable,
        _oracle_retrieve,
    )
    want = expected(g)
    assert len(got) == len(want)
    for i, (a, b) in enumerate(zip(got, want)):
        # decisions AND the float64 similarity are bit-identical to the reference
        assert a == b, (name, i, a, b)


@pytest.mark.parametrize(
    "sim,expected_k",
    [(0.305, 30), (0.265, 10), (1.0, 30), (0.25, 5), (0.2499999, None), (-1.0, None)],
)
def test_select_k_kat(sim, expected_k):  # test_cache.py:83-88
    assert OracleTable().select_k(sim) == expected_k


def test_select_k_monotone():  # test_cache.py:90-98
    t = OracleTable()
    prev = -1
    for s in np.linspace(-1, 1, 401):
        k = t.select_k(float(s))
        k = -1 if k is None else k
        assert k >= prev
        prev = k


def test_scan_oracle_agrees_with_store_oracle():
    rng = np.random.default_rng(4242)
    c = OracleCache(500, 32)
    for i in range(700):
        v = rng.standard_normal(32)
        c.insert(OracleEntry(f"e{i}", v / np.linalg.norm(v), "large", i, float(i)))
    m = np.stack([e.embedding for e in c.meta])
    t = OracleTable()
    for _ in range(200):
        q = rng.standard_normal(32)
        q /= np.linalg.norm(q)
        live, sim, k = c.retrieve(q, t)
        live2, sim2, k2, _ = scan_oracle(m, q, t)
        assert (live, k) == (live2, k2)
        assert abs(sim - sim2) <= 1e-15
