"""Device timeline of the pipelined C2 request loop (two lookups in flight, no inserts) from
torch.profiler (CUPTI): kernel start/duration and the host's submit/wait calls."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2503_11972_b200 import CacheEntry, SemanticCache, ThresholdTable  # noqa: E402

n, dim = 100_000, 768
rows, Q, new = bench.make_workload(dim, n, 1000)
c = SemanticCache(capacity=n, dim=dim)
c.bulk_load(CacheEntry(f"e{i}", rows[i], "large", i, 0.0) for i in range(n))
t = ThresholdTable.default()
ring = c.ring
c.retrieve(Q[0], t)


def raw(first, count):
    prev = None
    for i in range(first, first + count):
        tk = ring.submit1(Q[i])
        if prev is not None:
            ring.wait1(prev)
        prev = tk
    ring.wait1(prev)


raw(1, 200)
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    raw(300, 60)
rows_ = []
for e in prof.events():
    if e.device_type.name == "CUDA":
        rows_.append((e.time_range.start, e.time_range.end, "GPU", e.name[:50]))
    elif e.name in ("cudaLaunchKernelExC", "cudaLaunchKernel", "cudaMemcpyAsync"):
        rows_.append((e.time_range.start, e.time_range.end, "CPU", e.name))
rows_.sort()
t0 = rows_[0][0]
for s, e, kind, nm in rows_[-40:]:
    print(f"{s - t0:10.1f} {e - s:7.1f} {kind} {nm}")
