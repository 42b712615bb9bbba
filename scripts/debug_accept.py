"""Replay test_acceptance.py:411-443's workload (dim 32, 10k entries, seed 4242) on the GPU cache
and print every lookup whose entry differs from numpy's linear scan, with exact similarities
(fractions) of both rows.  Diagnostic only."""
import sys
from fractions import Fraction
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_11972_b200 import CacheEntry, SemanticCache, ThresholdTable  # noqa: E402
from paper_2503_11972_b200.records import normalize  # noqa: E402


def exact(a, b):
    return sum(Fraction(float(x)) * Fraction(float(y)) for x, y in zip(a, b))


dim = 32
rng = np.random.default_rng(4242)
cache = SemanticCache(capacity=10000, dim=dim)
for i in range(10000):
    cache.insert(CacheEntry(f"e{i}", normalize(rng.standard_normal(dim)), "large", i, float(i)))
table = ThresholdTable.default()
entries = cache.entries()
matrix = np.stack([e.embedding for e in entries])
bad = 0
for t in range(10000):
    q = normalize(rng.standard_normal(dim))
    got = cache.retrieve(q, table)
    sims = matrix @ q
    best = float(sims.max())
    bi = int(np.flatnonzero(sims == best)[-1])
    gi = int(got.entry.id[1:]) if got.hit else None
    if best >= 0.25 and gi != bi:
        bad += 1
        eb, eg = exact(matrix[bi], q), (exact(matrix[gi], q) if gi is not None else None)
        print(f"q{t}: numpy e{bi} {best!r}  gpu e{gi} {got.similarity!r} k={got.k}  "
              f"exact numpy-row {float(eb)!r} gpu-row {float(eg) if eg is not None else None!r} "
              f"exact diff {float(eg - eb) if eg is not None else None!r}  flags={cache.retrieve_flags(q[None], table)}")
        if bad > 10:
            break
print("mismatches", bad)
