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
# the bench's e2e step: async lookup, the insert while the scan runs, then the result
t0 = time.perf_counter()
for i in range(iters):
    pend = c.retrieve_async(Q[i], t)
    c.add(f"a{i}", imgs[i], "large", 1.0 + iters + i)
    pend.result()
t1 = time.perf_counter()
print(f"public API retrieve_async + add + result: {1e6 * (t1 - t0) / iters:.1f} us")
# pieces on the host: submit alone (wait right after), add alone, result alone
ts = ta = tr = 0.0
for i in range(iters):
    a0 = time.perf_counter()
    pend = c.retrieve_async(Q[i], t)
    a1 = time.perf_counter()
    c.add(f"b{i}", imgs[i], "large", 1.0 + 2 * iters + i)
    a2 = time.perf_counter()
    time.sleep(0)  # let the scan finish before timing result()
    while False:
        pass
    a3 = time.perf_counter()
    pend.result()
    a4 = time.perf_counter()
    ts += a1 - a0
    ta += a2 - a1
    tr += a4 - a3
print(f"host pieces: retrieve_async {1e6 * ts / iters:.1f} us, add {1e6 * ta / iters:.1f} us, "
      f"result (incl. waiting) {1e6 * tr / iters:.1f} us")
# pipelined (the bench's headline loop): submit i+1, insert, then the answer of i
ts = ta = tr = 0.0
prev = None
t0 = time.perf_counter()
for i in range(iters):
    a0 = time.perf_counter()
    pend = c.retrieve_async(Q[i], t)
    a1 = time.perf_counter()
    c.add(f"p{i}", imgs[i], "large", 1.0 + 3 * iters + i)
    a2 = time.perf_counter()
    if prev is not None:
        prev.result()
    a3 = time.perf_counter()
    prev = pend
    ts += a1 - a0
    ta += a2 - a1
    tr += a3 - a2
prev.result()
t1 = time.perf_counter()
print(f"pipelined: {1e6 * (t1 - t0) / iters:.1f} us per request; retrieve_async {1e6 * ts / iters:.1f} us, "
      f"add {1e6 * ta / iters:.1f} us, previous result (incl. waiting) {1e6 * tr / iters:.1f} us")
