# fp16 CTA-pair scan bisection (C3), kernel time from ncu launch lists:
# 1 no TMA, 2 no MMA, 4 no epilogue, 8 ring tiles t&7 (L2-resident ring)
mkdir -p gpurun_out
for d in ${DBGS:-0 4 6 5 8 12 7}; do
  MC_TC_DEBUG=$d timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tc_scan|k_tc8_scan" -c 10 \
    --csv --log-file gpurun_out/tcl$d.csv python scripts/tc_bisect.py ${TCP:-gemm} >/dev/null 2>&1
  echo "dbg=$d $(python scripts/ncu_times.py gpurun_out/tcl$d.csv)"
done
