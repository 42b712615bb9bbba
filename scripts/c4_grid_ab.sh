#!/usr/bin/env bash
# Sharded-path local lookups (pipelined, one GPU, one shard) with the streamed scan's wide grid
# (every co-resident CTA slot) vs the overlap grid, at a 1M window (C4 unsharded) and a 125k
# window (one shard of C4 at G = 8).  Output: gpurun_out/c4_grid_ab.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for wide in 0 1000000000000; do
MC_S8_WIDE_ROWS=$wide python - <<'PY'
import json, os, bench
for n in (1_000_000, 125_000):
    r = bench.run_sharded_c4(None, n, 1, 400, 20)
    print(f"wide_rows={os.environ['MC_S8_WIDE_ROWS']:>14} n={n:>8} B=1 step {1e3 * r['ms_per_step']:.1f} us  {r['value']:.0f}/s")
PY
done; done > gpurun_out/c4_grid_ab.log 2>&1
