"""Host-side profile of the C2 pipelined e2e loop (measurement tooling, GPU box): cProfile of
3000 requests (retrieve_async, add, previous .result()), top functions by own time."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2503_11972_b200 import CacheEntry, SemanticCache, ThresholdTable  # noqa: E402

n, dim, N = 100_000, 768, 3000
rows, Q, new = bench.make_workload(dim, n, 2 * N + 400)
c = SemanticCache(capacity=n, dim=dim)
c.bulk_load(CacheEntry(f"e{i}", rows[i], "large", i, 0.0) for i in range(n))
t = ThresholdTable.default()


def loop(first, count):
    prev = None
    for i in range(first, first + count):
        pend = c.retrieve_async(Q[i], t)
        c.add(f"s{i}", new[i], "large", 1000.0 + i)
        if prev is not None:
            prev.result()
        prev = pend
    prev.result()


loop(0, 400)
t0 = time.perf_counter()
loop(400, N)
print(f"plain: {1e6 * (time.perf_counter() - t0) / N:.2f} us per request")
pr = cProfile.Profile()
pr.enable()
loop(400 + N, N)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
