"""C3 tensor-core scan timing per path (measurement tooling): per-step events, L2 flushed between steps.
    MC_TC8_DEBUG / MC_TC_DEBUG bisection switches are read when the plan is created."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_11972_b200 import ThresholdTable, _native  # noqa: E402
from paper_2503_11972_b200.workload import ClusteredWorkload  # noqa: E402

path = {"gemm": 2, "gemm8": 7}[sys.argv[1]]
n, dim, B = 100_000, 1024, 256
wl = ClusteredWorkload(dim, n_clusters=512, seed=17)
ring = _native.DeviceRing(n, dim, 0)
ring.append(wl.cache_rows(n))
t = ThresholdTable.default()
ring.set_table(t.pairs, t.total_steps)
ring.set_path(path)
Q = wl.queries(B * 20).reshape(20, B, dim)
p = ring.profile_steps(Q, None, 20, 256 << 20)
print(sys.argv[1], "scan %.1f us  merge %.1f us  step %.1f us  fallback-steps %d" % (
    1e3 * p["scan_ms"], 1e3 * p["merge_ms"], 1e3 * p["step_ms"], p["would_fallback"]))
