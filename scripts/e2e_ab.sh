# e2e A/B on one box: the public-API request loop (retrieve_async + add + result) with the
# default envelope H2D vs MC_PARAM_INPUT=1 (inputs in the launch parameter block).
for r in 1 2; do
  for pi in 0 1; do
    MC_PARAM_INPUT=$pi MC_HOST_TIMING=1 timeout 300 python scripts/e2e_breakdown.py > gpurun_out/e2e_$pi.log 2>&1
    echo "param_in=$pi: $(grep -E 'retrieve_async \+ add|host pieces|host timing' gpurun_out/e2e_$pi.log | tr '\n' ' ')"
  done
done
