mkdir -p gpurun_out/ncu8
ncu --set full --clock-control none --import-source on -k regex:k_tc8_scan_pair -s 2 -c 1 -o gpurun_out/ncu8/tc8_c3 \
    python scripts/profile_case.py c3 --iters 4 --path gemm8 > gpurun_out/ncu8/tc8.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_merge8 -s 2 -c 1 -o gpurun_out/ncu8/merge8_c3 \
    python scripts/profile_case.py c3 --iters 4 --path gemm8 > gpurun_out/ncu8/merge8.log 2>&1
tail -2 gpurun_out/ncu8/tc8.log
