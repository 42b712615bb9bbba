timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
MC_HOST_TIMING=1 python scripts/e2e_breakdown.py 2>&1 | tail -5
SECONDS=0; timeout 900 python bench.py --no-c3 --cpu-seconds 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$? wall=$SECONDS
