"""C2 pipelined request floor (measurement tooling, GPU box): the same 100k x 768 cache driven by
(a) the public API (retrieve_async, add, previous .result()), (b) the DeviceRing calls alone
(submit1, append1, previous wait1) and (c) submit1 + wait1 without inserts -- per-request times."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2503_11972_b200 import CacheEntry, SemanticCache, ThresholdTable  # noqa: E402

n, dim, N = 100_000, 768, 3000
rows, Q, new = bench.make_workload(dim, n, 4 * N + 400)
c = SemanticCache(capacity=n, dim=dim)
c.bulk_load(CacheEntry(f"e{i}", rows[i], "large", i, 0.0) for i in range(n))
t = ThresholdTable.default()


def api(first, count):
    prev = None
    for i in range(first, first + count):
        pend = c.retrieve_async(Q[i], t)
        c.add(f"s{i}", new[i], "large", 1000.0 + i)
        if prev is not None:
            prev.result()
        prev = pend
    prev.result()


api(0, 300)
t0 = time.perf_counter()
api(300, N)
print(f"(a) public API: {1e6 * (time.perf_counter() - t0) / N:.2f} us per request")
ring = c.ring


def raw(first, count, insert):
    prev = None
    for i in range(first, first + count):
        tk = ring.submit1(Q[i])
        if insert:
            ring.append1(new[i])
        if prev is not None:
            ring.wait1(prev)
        prev = tk
    ring.wait1(prev)


c._settle()
for label, ins, off in (("(b) ring submit1 + append1 + wait1", True, 300 + N), ("(c) ring submit1 + wait1", False, 300 + 2 * N)):
    raw(off - 100, 100, ins)
    t0 = time.perf_counter()
    raw(off, N, ins)
    print(f"{label}: {1e6 * (time.perf_counter() - t0) / N:.2f} us per request")

# (d) where the host time goes in (c): the submit call and the wait call, timed separately
ts = tw = 0.0
prev = None
off = 300 + 3 * N
for i in range(off, off + N):
    a = time.perf_counter()
    tk = ring.submit1(Q[i])
    b = time.perf_counter()
    if prev is not None:
        ring.wait1(prev)
    e = time.perf_counter()
    ts += b - a
    tw += e - b
    prev = tk
ring.wait1(prev)
print(f"(d) submit1 {1e6 * ts / N:.2f} us, wait1 {1e6 * tw / N:.2f} us per request")
