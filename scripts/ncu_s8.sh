# one full ncu capture of the streamed int8 scan (C2) with source-level stall sampling
mkdir -p gpurun_out/ncu
ncu --set full --clock-control none --import-source on -k regex:k_stream8_scan -s 3 -c 1 -o gpurun_out/ncu/s8_c2 \
    python scripts/profile_case.py c2 --iters 5 > gpurun_out/ncu/s8.log 2>&1
echo ncu rc=$?
tail -3 gpurun_out/ncu/s8.log
ls -la gpurun_out/ncu
