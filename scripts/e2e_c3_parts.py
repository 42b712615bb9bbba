"""C3 end-to-end parts with the batch taken from a page-locked array (measurement tooling, GPU box):
native batched call, public retrieve_batch, and a bare 2 MB H2D copy of the same bytes."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_11972_b200 import CacheEntry, SemanticCache, ThresholdTable  # noqa: E402
from paper_2503_11972_b200.workload import ClusteredWorkload  # noqa: E402

n, dim, B, iters = 100_000, 1024, 256, 100
wl = ClusteredWorkload(dim, n_clusters=512, seed=17)
rows = wl.cache_rows(n)
Q = np.ascontiguousarray(wl.queries(B * (iters + 2)).reshape(iters + 2, B, dim))
c = SemanticCache(capacity=n, dim=dim)
c.ring.append(rows)
c._store.extend(CacheEntry(f"e{i}", rows[i], "large", i, 0.0) for i in range(n))
c._next_seq = n
t = ThresholdTable.default()
c.register_host_buffer(Q)
c.retrieve_batch(Q[0], t)
for label, fn in (("native ring.retrieve", lambda i: c.ring.retrieve(Q[i])),
                  ("public retrieve_batch", lambda i: c.retrieve_batch(Q[i], t))):
    fn(1)
    t0 = time.perf_counter()
    for i in range(iters):
        fn(1 + i)
    print(f"{label}: {1e6 * (time.perf_counter() - t0) / iters:.1f} us per batch")
Qt = torch.from_numpy(Q)
dst = torch.empty(B * dim, dtype=torch.float64, device="cuda")
for _ in range(3):
    dst.copy_(Qt[1].reshape(-1), non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(iters):
    dst.copy_(Qt[1 + i].reshape(-1), non_blocking=True)
    torch.cuda.synchronize()
print(f"bare 2 MB H2D from page-locked memory + sync: {1e6 * (time.perf_counter() - t0) / iters:.1f} us")
st = c.ring.stats()
print(st)
