# Pair-kernel cycle accounting at C3 for the full kernel and the MMA-only / TMA-only bisections.
for dbg in 0 5 6 4; do
  MC_GEMV_TIMING=1 MC_TC_DEBUG=$dbg timeout 300 python scripts/tc_timers.py
done
