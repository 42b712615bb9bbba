for n in 2000 20000 50000 100000 200000; do for d in 7 0; do
  MC_TC_DEBUG=$d ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bn.csv python scripts/profile_case.py c3 --iters 3 --entries $n > /dev/null 2>&1
  echo "n=$n dbg=$d $(grep k_tc_scan gpurun_out/bn.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done; done
