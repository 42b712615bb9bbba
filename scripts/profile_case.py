"""Drive one BASELINE config through the native ring for ncu / timing (no oracle, no host metadata).

    python scripts/profile_case.py c2|c3 [--iters N] [--path auto|gemv|gemm|stream8] [--rotate K]

--rotate K: K rings with the same contents, lookup i on ring i % K (K x the scan copy > L2: cold HBM
reads every lookup, as in bench.py's rotation).
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
ap.add_argument("--rotate", type=int, default=1)
a = ap.parse_args()
n, dim, B = CASES[a.case]
B = a.batch or B
n = a.entries or n
wl = ClusteredWorkload(dim, n_clusters=512, seed=17)
rows = wl.cache_rows(n)
rings = []
t = ThresholdTable.default()
for _ in range(a.rotate):
    ring = _native.DeviceRing(n, dim, 0)
    ring.append(rows)
    ring.set_path({"auto": 0, "gemv": 1, "gemm": 2, "stream8": 6}[a.path])
    ring.set_table(t.pairs, t.total_steps)
    rings.append(ring)
ring = rings[0]
Q = wl.queries(B * a.iters).reshape(a.iters, B, dim)
for i in range(a.iters):
    live, sim, k, flags = rings[i % a.rotate].retrieve(Q[i])
print(a.case, "ok", ring.stats())

import os  # noqa: E402
if os.environ.get("MC_GEMV_TIMING"):
    import ctypes  # noqa: E402
    lib = _native.load()
    lib.mc_debug_gemv_timing.restype = ctypes.c_int
    t = (ctypes.c_ulonglong * 8)()
    per = (ctypes.c_ulonglong * (12 * 512))()
    for i in range(a.iters):
        lib.mc_debug_gemv_timing(t, 1)  # reset
        ring = rings[i % a.rotate]
        ring.retrieve(Q[i])
        lib.mc_debug_gemv_timing(t, 0)
        if not t[4]:  # register GEMV kernels: four global stamps
            print("gemv phases (us): scan %.1f  rescore %.1f  tail %.1f  total %.1f" % (
                (t[1] - t[0]) / 1e3, (t[2] - t[1]) / 1e3, (t[3] - t[2]) / 1e3, (t[3] - t[0]) / 1e3))
            continue
        lib.mc_debug_gemv_timing(per, 2)
        import numpy as _np
        arr = _np.array(per[:8 * 148], dtype=_np.float64).reshape(148, 8)
        t0 = float(t[0])
        rel = lambda v: (v - t0) / 1e3  # noqa: E731
        scan_end, pool, r0, r1, poolx, rec = (arr[:, k] for k in range(6))
        r0 = _np.where(r0 > 1e19, _np.nan, r0)
        print("stream8 (us): last scan end %.1f | last record %.1f | ticket->merge %.1f loads %.1f decide %.1f | total %.1f"
              " | pushed %d rescored %d" % (rel(scan_end.max()), rel(rec.max()), (t[4] - rec.max()) / 1e3,
                                             (t[5] - t[4]) / 1e3, (t[3] - t[5]) / 1e3, rel(t[3]),
                                             arr[:, 6].sum(), arr[:, 7].sum()))
        if t[6] and t[7]:
            print("   tail detail (us): reductions %.2f | record+decide+result store %.2f | rest %.2f" % (
                (t[6] - t[5]) / 1e3, (t[7] - t[6]) / 1e3, (t[3] - t[7]) / 1e3))
        if i == a.iters - 1:
            order = _np.argsort(-rec)
            cyc = _np.array(per[8 * 512:8 * 512 + 4 * 148], dtype=_np.float64).reshape(148, 4)
            print("slowest CTAs: cta scan_end pool_entry resc_start resc_end pool_exit record n_resc (us) | "
                  "cycles: first_pass second_pass first_dot dot")
            for c in order[:8]:
                print("   %4d %6.1f %6.1f %6.1f %6.1f %6.1f %6.1f %3d | %6d %4d %6d %6d" % (
                    c, rel(scan_end[c]), rel(pool[c]), rel(r0[c]), rel(r1[c]) if r1[c] else _np.nan, rel(poolx[c]),
                    rel(rec[c]), arr[c, 7], cyc[c, 0], cyc[c, 1], cyc[c, 2] if cyc[c, 2] < 1e18 else -1, cyc[c, 3]))
            print("median: scan_end %.1f pool_entry %.1f pool_exit %.1f record %.1f" % (
                rel(_np.median(scan_end)), rel(_np.median(pool)), rel(_np.median(poolx)), rel(_np.median(rec))))
