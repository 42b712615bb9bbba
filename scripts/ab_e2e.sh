#!/usr/bin/env bash
# e2e A/B of library builds (MODMCACHE_LIB): C2 and C1 pipelined / one-at-a-time request loops.
#   LIBS="a.so b.so" (paths under paper_2503_11972_b200/); output on stdout
cd "$(dirname "$0")/.."
for r in 1 2; do for lib in $LIBS; do
MODMCACHE_LIB=paper_2503_11972_b200/$lib timeout 300 python - <<PY 2>/dev/null | grep '^lib'
import bench
pk = bench.peaks()
for name, n, rot in (("c2", 100_000, 4), ("c1", 10_000, 1)):
    r = bench.run_config(name, 768, n, 1, 500, 5, True, (256 << 20) if rot > 1 else 0, pk, n_rot=rot, e2e_steps=3000)
    print("lib $lib %s step %.2f us e2e %.0f/s (%.1f us) seq %.0f/s (%.1f us)" % (name, 1e3*r["ms_per_step"], r["e2e"]["value"], r["e2e"]["latency_us"], r["e2e"]["sequential"]["value"], r["e2e"]["sequential"]["latency_us"]))
PY
done; done
