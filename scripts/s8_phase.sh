MC_GEMV_TIMING=1 timeout 120 python scripts/profile_case.py c2 --iters 8 > gpurun_out/phases.log 2>&1; echo phases rc=$?
tail -8 gpurun_out/phases.log
MC_GEMV_TIMING=1 timeout 120 python scripts/profile_case.py c1 --iters 4 > gpurun_out/phases_c1.log 2>&1; tail -4 gpurun_out/phases_c1.log
