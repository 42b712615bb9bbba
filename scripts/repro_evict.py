"""Minimal reproduction attempt: pending appends interleaved with multi-row age evictions."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_11972_b200 import CacheEntry, SemanticCache, ThresholdTable  # noqa: E402

check_path = int(sys.argv[1])
lookup_path = int(sys.argv[2])
rng = np.random.default_rng(7)
dim, cap = 96, 603
c = SemanticCache(capacity=cap, dim=dim, max_age_s=100.0)
table = ThresholdTable.default()
t = 0.0
seq = 0


def emb():
    v = rng.standard_normal(dim)
    return v / np.linalg.norm(v)


def check(tag):
    M = np.stack([x.embedding for x in c.entries()])
    c.ring.set_path(check_path)
    l, s, k, f = c.retrieve_flags(M, table)
    bad = [i for i in range(len(M)) if abs(s[i] - 1) > 1e-9]
    if bad:
        print("BAD after", tag, "live", len(M), bad[:8])
        return False
    return True


for rnd in range(40):
    n = int(rng.integers(1, 30))
    for j in range(n):
        t += float(rng.exponential(0.5)) + (float(rng.integers(2, 8)) if rng.random() < 0.1 else 0.0)
        c.insert(CacheEntry(f"e{seq}", emb(), "large", seq, t))
        seq += 1
    if rng.random() < 0.5:  # a small lookup on the path under test
        c.ring.set_path(lookup_path)
        B = int(rng.choice([1, 2, 4, 17]))
        c.retrieve_batch(np.stack([emb() for _ in range(B)]), table)
    if not check(f"round {rnd}"):
        break
else:
    print("ok", check_path, lookup_path, "live", len(c))
