"""C3 tensor-core scan timing per path (measurement tooling).  Prints the back-to-back step time
(rotation over 2 caches, together > L2) and the scan / merge split of isolated warm steps.
MC_TC8_DEBUG / MC_TC_DEBUG bisection switches are read when the plan is created."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_11972_b200 import ThresholdTable, _native  # noqa: E402
from paper_2503_11972_b200.workload import ClusteredWorkload  # noqa: E402

path = {"gemm": 2, "gemm8": 7, "quad": 4}[sys.argv[1]]
import os
n, dim, B = int(os.environ.get("TC_N", 100_000)), 1024, int(os.environ.get("TC_B", 256))
wl = ClusteredWorkload(dim, n_clusters=512, seed=17)
t = ThresholdTable.default()
rings = []
for i in range(2):
    ring = _native.DeviceRing(n, dim, 0)
    ring.append(wl.cache_rows(n))
    ring.set_table(t.pairs, t.total_steps)
    ring.set_path(path)
    rings.append(ring)
Q = wl.queries(B * 40).reshape(40, B, dim)
for _ in range(2):
    r = _native.DeviceRing.profile_rotate(rings, Q, None, 40)
p = rings[0].profile_steps(Q[:20], None, 20, 0)
print(sys.argv[1], "rotate step %.1f us | warm isolated: scan %.1f us  merge %.1f us  fallback-steps %d" % (
    1e3 * r["step_ms"], 1e3 * p["scan_ms"], 1e3 * p["merge_ms"], p["would_fallback"]))
