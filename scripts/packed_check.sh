timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_gpu.log
MC_PACKED_RESULT=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "async or fifo or golden or smoke or config2" > gpurun_out/pytest_gpu_fenced.log 2>&1; echo pytest-fenced rc=$?; tail -1 gpurun_out/pytest_gpu_fenced.log
MC_HOST_TIMING=1 python scripts/e2e_breakdown.py 2>&1 | tail -5
SECONDS=0; timeout 900 python bench.py --no-c3 --cpu-seconds 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$? wall=$SECONDS
