# stream8 bring-up: smoke, GPU parity, phase timing, short bench (outputs in gpurun_out/)
set -x
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -5 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -x -rA ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|Error|error" gpurun_out/pytest_gpu.log | tail -15
MC_GEMV_TIMING=1 timeout 120 python scripts/profile_case.py c2 --iters 8 > gpurun_out/phases.log 2>&1; echo phases rc=$?
tail -9 gpurun_out/phases.log
MC_GEMV_TIMING=1 timeout 120 python scripts/profile_case.py c2 --iters 8 --path gemv8 > gpurun_out/phases8.log 2>&1
tail -4 gpurun_out/phases8.log
timeout 600 python bench.py --steps ${BENCH_STEPS:-200} --warmup 5 --cpu-seconds 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -3 gpurun_out/bench.err
