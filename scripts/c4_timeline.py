"""Device timeline of pipelined sharded C4 steps (one GPU, one shard) from torch.profiler (CUPTI):
kernels and copies with their start/end, to find where a step's time goes beyond the scan."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
bench.run_sharded_c4(None, 1_000_000, B, 20, 5)  # warm everything
_orig = torch.cuda.Event


with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    r = bench.run_sharded_c4(None, 1_000_000, B, 12, 3)
print(json.dumps({k: r[k] for k in ("value", "ms_per_step")}))
evs = [e for e in prof.events() if e.device_type.name == "CUDA" or "cuda" in e.name.lower() or e.name.startswith("mc_")]
rows = []
for e in prof.events():
    if e.device_type.name == "CUDA":
        rows.append((e.time_range.start, e.time_range.end, "GPU", e.name[:60]))
    elif e.name.startswith("cuda") and e.name in ("cudaEventSynchronize", "cudaStreamSynchronize", "cudaMemcpyAsync",
                                                  "cudaLaunchKernel", "cudaLaunchKernelExC", "cudaStreamWaitEvent"):
        rows.append((e.time_range.start, e.time_range.end, "CPU", e.name))
rows.sort()
t0 = rows[0][0] if rows else 0
last = rows[-1][0] if rows else 0
for s, e, kind, n in rows:
    if s > last - 1500:  # the last ~1.5 ms
        print(f"{(s - t0):10.1f} {(e - s):8.1f} {kind} {n}")
