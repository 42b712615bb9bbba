# Launch list + full ncu capture of the scan kernels (one GPU).
set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python scripts/profile_case.py c3 --iters 4 > gpurun_out/ncu_c3_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tc_scan -s 2 -c 1 -o gpurun_out/prof_tc python scripts/profile_case.py c3 --iters 4 > gpurun_out/ncu_tc.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gemv_scan -s 2 -c 1 -o gpurun_out/prof_gemv python scripts/profile_case.py c2 --iters 4 > gpurun_out/ncu_gemv.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_merge -s 2 -c 1 -o gpurun_out/prof_merge python scripts/profile_case.py c2 --iters 4 > gpurun_out/ncu_merge.log 2>&1
ls -la gpurun_out
