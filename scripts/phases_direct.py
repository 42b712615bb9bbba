"""Phase stamps (MC_GEMV_TIMING=1) of the single-query direct lookup (retrieve1: the path the
public API takes), with or without MC_PARAM_INPUT=1.  Diagnostic only."""
import ctypes
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_11972_b200 import ThresholdTable, _native  # noqa: E402
from paper_2503_11972_b200.workload import ClusteredWorkload  # noqa: E402

n, dim = 100_000, 768
wl = ClusteredWorkload(dim, n_clusters=512, seed=17)
ring = _native.DeviceRing(n, dim, 0)
ring.append(wl.cache_rows(n))
t = ThresholdTable.default()
ring.set_table(t.pairs, t.total_steps)
Q = wl.queries(64)
imgs = wl.images(Q)
lib = _native.load()
g = (ctypes.c_ulonglong * 8)()
per = (ctypes.c_ulonglong * (12 * 512))()
res = []
for i in range(40):
    ring.append1(imgs[i])  # one pending row per lookup, as in the e2e loop
    lib.mc_debug_gemv_timing(g, 1)
    ring.retrieve1(Q[i])
    lib.mc_debug_gemv_timing(g, 0)
    lib.mc_debug_gemv_timing(per, 2)
    arr = np.array(per[:8 * 148], dtype=np.float64).reshape(148, 8)
    t0 = float(g[0])
    res.append([(arr[:, 0].max() - t0) / 1e3, (np.median(arr[:, 0]) - t0) / 1e3, (arr[:, 5].max() - t0) / 1e3,
                (float(g[3]) - t0) / 1e3, (arr[0, 5] - t0) / 1e3])
r = np.median(np.array(res[5:]), axis=0)
print("median over lookups (us from first CTA start): last scan end %.1f | median scan end %.1f | last record %.1f | "
      "decision %.1f | CTA0 record %.1f" % tuple(r))
order = np.argsort(-arr[:, 5])
print("slowest CTAs of the last lookup (us): cta scan_end pool_entry resc_start resc_end pool_exit record n_resc")
for c in order[:10]:
    v = arr[c]
    f = lambda x: (x - t0) / 1e3 if 0 < x < 1.8e19 else float("nan")  # noqa: E731
    print("   %4d %6.1f %6.1f %6.1f %6.1f %6.1f %6.1f %3d" % (c, f(v[0]), f(v[1]), f(v[2]), f(v[3]), f(v[4]), f(v[5]), v[7]))
print("records landed by (us): p50 %.1f p90 %.1f max %.1f; rescored per CTA: mean %.2f max %d" % (
    (np.median(arr[:, 5]) - t0) / 1e3, (np.percentile(arr[:, 5], 90) - t0) / 1e3, (arr[:, 5].max() - t0) / 1e3,
    arr[:, 7].mean(), arr[:, 7].max()))
