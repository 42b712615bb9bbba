set -x
timeout 600 python -m pytest tests -m gpu -q -x -k "tensor_core or duplicates or clustered" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python scripts/profile_case.py c3 --iters 4 > /dev/null 2>&1
grep -E "k_tc_scan|k_merge" gpurun_out/launches_c3.csv | awk -F'","' '{print $5, $NF}' | cut -c1-40,100-
ncu --set full --clock-control none --import-source on -k regex:k_tc_scan -s 2 -c 1 -o gpurun_out/prof_tc python scripts/profile_case.py c3 --iters 4 > gpurun_out/ncu_tc.log 2>&1
