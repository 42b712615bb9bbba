"""Drive one BASELINE config through the native ring for ncu / timing (no oracle, no host metadata).

    python scripts/profile_case.py c2|c3 [--iters N] [--path auto|gemv|gemm]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_11972_b200 import ThresholdTable, _native  # noqa: E402
from paper_2503_11972_b200.workload import ClusteredWorkload  # noqa: E402

CASES = {"c1": (10_000, 768, 1), "c2": (100_000, 768, 1), "c3": (100_000, 1024, 256)}

ap = argparse.ArgumentParser()
ap.add_argument("case", choices=sorted(CASES))
ap.add_argument("--iters", type=int, default=6)
ap.add_argument("--path", default="auto")
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--entries", type=int, default=0)
a = ap.parse_args()
n, dim, B = CASES[a.case]
B = a.batch or B
n = a.entries or n
wl = ClusteredWorkload(dim, n_clusters=512, seed=17)
rows = wl.cache_rows(n)
ring = _native.DeviceRing(n, dim, 0)
ring.append(rows)
ring.set_path({"auto": 0, "gemv": 1, "gemm": 2}[a.path])
t = ThresholdTable.default()
ring.set_table(t.pairs, t.total_steps)
Q = wl.queries(B * a.iters).reshape(a.iters, B, dim)
for i in range(a.iters):
    live, sim, k, flags = ring.retrieve(Q[i])
print(a.case, "ok", ring.stats())

import os  # noqa: E402
if os.environ.get("MC_GEMV_TIMING"):
    import ctypes  # noqa: E402
    lib = _native.load()
    lib.mc_debug_gemv_timing.restype = ctypes.c_int
    t = (ctypes.c_ulonglong * 4)()
    for i in range(a.iters):
        lib.mc_debug_gemv_timing(t, 1)  # reset
        ring.retrieve(Q[i])
        lib.mc_debug_gemv_timing(t, 0)
        print("gemv phases (us): scan %.1f  rescore %.1f  tail %.1f  total %.1f" % (
            (t[1] - t[0]) / 1e3, (t[2] - t[1]) / 1e3, (t[3] - t[2]) / 1e3, (t[3] - t[0]) / 1e3))
