# Round-2 ncu evidence (one GPU, never multi-rank): launch list of the bench command, then one
# --set full capture per top kernel.  Reports land in gpurun_out/ncu/ and are summarised into
# profiles/ in the build container (scripts/ncu_summary.py).
set -x
mkdir -p gpurun_out/ncu
rm -f gpurun_out/ncu/*.ncu-rep
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches_bench.csv \
    python bench.py --steps 8 --warmup 3 --cpu-seconds 0.2 --no-big > gpurun_out/ncu/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stream8_scan -s 3 -c 1 -o gpurun_out/ncu/s8_c2 \
    python scripts/profile_case.py c2 --iters 5 --rotate 4 > gpurun_out/ncu/s8.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tc_scan_pair -s 2 -c 1 -o gpurun_out/ncu/tc_pair_c3 \
    python scripts/profile_case.py c3 --iters 4 --rotate 2 > gpurun_out/ncu/tc.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_merge -s 2 -c 1 -o gpurun_out/ncu/merge_c3 \
    python scripts/profile_case.py c3 --iters 4 --rotate 2 > gpurun_out/ncu/merge.log 2>&1
ls -la gpurun_out/ncu
