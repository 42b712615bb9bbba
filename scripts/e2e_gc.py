"""Does Python's cyclic GC show up in the public-API request loop?  Same loop with gc enabled,
gc.freeze()'d after setup, and disabled (measurement only)."""
import gc
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_11972_b200 import CacheEntry, SemanticCache, ThresholdTable  # noqa: E402
from paper_2503_11972_b200.workload import ClusteredWorkload  # noqa: E402

n, dim, iters = 100_000, 768, 3000
wl = ClusteredWorkload(dim, n_clusters=512, seed=17)
rows = wl.cache_rows(n)
Q = wl.queries(4 * iters + 400)
imgs = wl.images(Q)
c = SemanticCache(capacity=n, dim=dim)
c.bulk_load(CacheEntry(f"e{i}", rows[i], "large", i, 0.0) for i in range(n))
t = ThresholdTable.default()
j = 0
for mode in ("enabled", "frozen", "disabled", "enabled"):
    if mode == "frozen":
        gc.collect()
        gc.freeze()
    if mode == "disabled":
        gc.disable()
    if mode == "enabled":
        gc.enable()
        gc.unfreeze()
    for i in range(50):
        p = c.retrieve_async(Q[j], t); c.add(f"w{j}", imgs[j], "large", 1.0 + j); p.result(); j += 1
    t0 = time.perf_counter()
    for i in range(iters):
        p = c.retrieve_async(Q[j], t)
        c.add(f"s{j}", imgs[j], "large", 1.0 + j)
        p.result()
        j += 1
    dt = time.perf_counter() - t0
    print(f"gc {mode:8s}: {1e6 * dt / iters:.1f} us per request ({iters / dt:.0f}/s); gc counts {gc.get_count()}")
