"""Does the launch's parameter-block size limit pipelined single-query lookups?  Raw submit1/wait1
loop (two in flight, no inserts) on a 100k x 256 cache; run once per library (MODMCACHE_LIB)."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2503_11972_b200 import CacheEntry, SemanticCache, ThresholdTable  # noqa: E402

n, dim, N = 100_000, int(sys.argv[1]) if len(sys.argv) > 1 else 256, 3000
rows, Q, new = bench.make_workload(dim, n, N + 400)
c = SemanticCache(capacity=n, dim=dim)
c.bulk_load(CacheEntry(f"e{i}", rows[i], "large", i, 0.0) for i in range(n))
c.retrieve(Q[0], ThresholdTable.default())
ring = c.ring


def raw(first, count):
    prev = None
    for i in range(first, first + count):
        tk = ring.submit1(Q[i])
        if prev is not None:
            ring.wait1(prev)
        prev = tk
    ring.wait1(prev)


raw(1, 300)
t0 = time.perf_counter()
raw(300, N)
print(f"{os.environ.get('MODMCACHE_LIB', 'default')} D={dim}: {1e6 * (time.perf_counter() - t0) / N:.2f} us per request")
