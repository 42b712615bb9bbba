"""C3 end-to-end pieces (measurement tooling, GPU box): native batched call vs the Python
result objects of retrieve_batch."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_11972_b200 import CacheEntry, SemanticCache, ThresholdTable  # noqa: E402
from paper_2503_11972_b200.workload import ClusteredWorkload  # noqa: E402

n, dim, B, iters = 100_000, 1024, 256, 50
wl = ClusteredWorkload(dim, n_clusters=512, seed=17)
rows = wl.cache_rows(n)
Q = wl.queries(B * (iters + 2)).reshape(iters + 2, B, dim)
c = SemanticCache(capacity=n, dim=dim)
c.ring.append(rows)
c._store.extend(CacheEntry(f"e{i}", rows[i], "large", i, 0.0) for i in range(n))
c._next_seq = n
t = ThresholdTable.default()
c.retrieve_batch(Q[0], t)
t0 = time.perf_counter()
for i in range(iters):
    c.ring.retrieve(Q[i + 1])
t1 = time.perf_counter()
print(f"native retrieve (B={B}): {1e6 * (t1 - t0) / iters:.1f} us per batch")
t0 = time.perf_counter()
for i in range(iters):
    c.retrieve_batch(Q[i + 1], t)
t1 = time.perf_counter()
print(f"public retrieve_batch: {1e6 * (t1 - t0) / iters:.1f} us per batch")
import os  # noqa: E402
os.environ.setdefault("MC_HOST_TIMING", "1")
import numpy as np  # noqa: E402
lib = c.ring.lib
# the pieces of one native batched call, from the library's host timers (printed at destroy)
Qc = np.ascontiguousarray(Q[1])
t0 = time.perf_counter()
for i in range(iters):
    np.copyto(Qc, Q[i + 1])
t1 = time.perf_counter()
print(f"host copy of a 2 MB float64 batch (numpy): {1e6 * (t1 - t0) / iters:.1f} us")
