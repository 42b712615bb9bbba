#!/usr/bin/env bash
# Single-query sharded-path local lookups: parameter-block launch (default) vs the envelope copy
# (MC_LOCAL_PARAM=0, wide grid), 1M and 125k windows.  Output: gpurun_out/c4_param_ab.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for prm in 1 0; do
MC_LOCAL_PARAM=$prm python - <<'PY'
import os, bench
for n in (1_000_000, 125_000):
    r = bench.run_sharded_c4(None, n, 1, 400, 20)
    print(f"local_param={os.environ['MC_LOCAL_PARAM']} n={n:>8} B=1 step {1e3 * r['ms_per_step']:.1f} us  {r['value']:.0f}/s")
PY
done; done > gpurun_out/c4_param_ab.log 2>&1
