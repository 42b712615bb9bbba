"""Where the C3 pair kernel's cycles go (measurement tooling, GPU box; needs MC_GEMV_TIMING=1):
per-cluster cycle sums recorded by k_tc_scan_pair (scan_tc.cu, `tim`), averaged per launch over
back-to-back C3 steps.  MC_TC_DEBUG switches apply (1 no TMA, 2 no MMA, 4 no epilogue)."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_11972_b200 import ThresholdTable, _native  # noqa: E402
from paper_2503_11972_b200.workload import ClusteredWorkload  # noqa: E402

assert os.environ.get("MC_GEMV_TIMING") == "1"
n, dim, B, iters = 100_000, 1024, 256, 40
wl = ClusteredWorkload(dim, n_clusters=512, seed=17)
t = ThresholdTable.default()
rings = []
for i in range(2):
    ring = _native.DeviceRing(n, dim, 0)
    ring.append(wl.cache_rows(n))
    ring.set_table(t.pairs, t.total_steps)
    rings.append(ring)
Q = wl.queries(B * iters).reshape(iters, B, dim)
lib = _native.load()
buf = np.zeros(12 * 512, dtype=np.uint64)
ptr = buf.ctypes.data_as(C.POINTER(C.c_double))
_native.DeviceRing.profile_rotate(rings, Q, None, iters)  # warm
lib.mc_debug_gemv_timing(ptr, 1)
r = _native.DeviceRing.profile_rotate(rings, Q, None, iters)
lib.mc_debug_gemv_timing(ptr, 2)
T = buf.reshape(512, 12).astype(np.float64)
launches = iters  # profile_rotate runs `iters` steps, one pair launch each
live = T[:, 3] > 0
T = T[live] / launches
names = ["MMA issue loop", "MMA wait full", "MMA wait tempty", "units", "producer wait empty",
         "epilogue wait tfull", "epilogue busy", "prologue"]
print(f"MC_TC_DEBUG={os.environ.get('MC_TC_DEBUG', '0')}: step {1e3 * r['step_ms']:.1f} us, {live.sum()} clusters")
ghz = T[:, 0].sum() / T[:, 8].sum()
print(f"  SM clock over the MMA-issue loops: {ghz:.2f} GHz; loop {T[:, 8].mean() / 1e3:.2f} us mean, "
      f"{T[:, 8].max() / 1e3:.2f} us max")
for i, nm in enumerate(names):
    v = T[:, i]
    unit = "" if i == 3 else f"  ({v.mean() / ghz / 1e3:6.2f} us)"
    print(f"  {nm:22s} mean {v.mean():10.0f}  max {v.max():10.0f}{unit}")
