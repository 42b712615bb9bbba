for d in ${DBGS:-0 6 14 8 7}; do
  MC_TC_DEBUG=$d ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bis_$d.csv python scripts/profile_case.py c3 --iters 3 > /dev/null 2>&1
  echo "dbg=$d $(grep k_tc_scan gpurun_out/bis_$d.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done
