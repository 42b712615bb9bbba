#!/usr/bin/env bash
# Streamed-scan grid sized by the window (MC_S8_ROWS_PER_CTA = rows per CTA, 0 = full grid):
# C1 (10k rows, L2-resident) and C2 (100k) back-to-back step, isolated lookup and e2e.
# Output: gpurun_out/s8_rows_ab.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for rpc in ${RPCS:-0 128 256 512}; do
MC_S8_ROWS_PER_CTA=$rpc python - <<'PY'
import os, bench
pk = bench.peaks()
for name, n, steps, e2e, rot in (("c1", 10_000, 1000, 1500, 1), ("c2", 100_000, 1000, 1500, 4)):
    r = bench.run_config(name, 768, n, 1, steps, 5, True, 256 << 20 if rot > 1 else 0, pk, n_rot=rot, e2e_steps=e2e)
    print(f"rows_per_cta={os.environ['MC_S8_ROWS_PER_CTA']:>4} {name}: back-to-back {1e3 * r['ms_per_step']:.2f} us, "
          f"isolated {1e3 * r['profile']['step_ms']:.2f} us, e2e {r['e2e']['value']:.0f}/s "
          f"(seq {r['e2e']['sequential']['value']:.0f}/s)")
PY
done; done > gpurun_out/s8_rows_ab.log 2>&1
