timeout 300 python -m pytest tests -m gpu -q -x -k "tensor_core or clustered or duplicates" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
for path in gemm gemm_pair_dummy; do :; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv timeout 120 python scripts/profile_case.py c3 --iters 4 > /dev/null 2>&1
grep -E "k_tc" gpurun_out/launches_c3.csv | awk -F'","' '{print $5, $NF}' | cut -c1-22,130-
