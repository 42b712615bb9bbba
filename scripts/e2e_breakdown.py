"""Where the end-to-end lookup time goes (measurement tooling, GPU box): kernel (warm L2),
native call (ctypes -> mc_retrieve_batch), and the public Python API with the FIFO insert."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_11972_b200 import CacheEntry, SemanticCache, ThresholdTable  # noqa: E402
from paper_2503_11972_b200.workload import ClusteredWorkload  # noqa: E402

n, dim, iters = 100_000, 768, 2000
wl = ClusteredWorkload(dim, n_clusters=512, seed=17)
rows = wl.cache_rows(n)
Q = wl.queries(iters + 10)
imgs = wl.images(Q)
c = SemanticCache(capacity=n, dim=dim)
c.ring.append(rows)
c._store.extend(CacheEntry(f"e{i}", rows[i], "large", i, 0.0) for i in range(n))
c._next_seq = n
t = ThresholdTable.default()
c.ring.set_table(t.pairs, t.total_steps)
prof = c.ring.profile_steps(Q[:200].reshape(200, 1, dim), None, 200, 0)
print(f"kernel (events, warm L2, no insert): {1e3 * prof['step_ms']:.1f} us")
prof = c.ring.profile_steps(Q[:200].reshape(200, 1, dim), imgs[:200], 200, 0)
print(f"kernel (events, warm L2, with insert): {1e3 * prof['step_ms']:.1f} us")
r = c.ring
for i in range(10):
    r.retrieve1(Q[i])
t0 = time.perf_counter()
for i in range(iters):
    r.retrieve1(Q[i])
t1 = time.perf_counter()
print(f"native retrieve1 (ctypes, no insert): {1e6 * (t1 - t0) / iters:.1f} us")
t0 = time.perf_counter()
for i in range(iters):
    r.retrieve1(Q[i])
    r.append1(imgs[i])
t1 = time.perf_counter()
print(f"native retrieve1 + append1: {1e6 * (t1 - t0) / iters:.1f} us")
t0 = time.perf_counter()
for i in range(iters):
    c.retrieve(Q[i], t)
    c.add(f"s{i}", imgs[i], "large", 1.0 + i)
t1 = time.perf_counter()
print(f"public API retrieve + add: {1e6 * (t1 - t0) / iters:.1f} us")
