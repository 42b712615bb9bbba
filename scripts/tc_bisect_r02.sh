# Pair-kernel bisection (ncu launch times of k_tc_scan_pair at C3, MC_TC_DEBUG switches):
# 0 full | 4 no epilogue | 2+4 TMA only (no MMA, no epilogue) | 8 ring tiles L2-resident | 1+4 MMA only (no TMA)
for dbg in 0 4 6 8 12 5; do
  MC_TC_DEBUG=$dbg ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_tc_scan_pair --csv \
      python scripts/profile_case.py c3 --iters 6 2>/dev/null | grep k_tc_scan_pair | tail -3 | \
      awk -F'","' -v d=$dbg '{gsub(/"/,"",$NF); s+=$NF; n++} END {printf "MC_TC_DEBUG=%-3s pair kernel %.1f us (mean of %d)\n", d, s/n/1000, n}'
done
