# One GPU round-trip: smoke, GPU parity suite, short bench.  Outputs land in gpurun_out/.
set -x
nvidia-smi -L
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests -m gpu -q -rA ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -40 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps ${BENCH_STEPS:-50} --warmup 5 --cpu-seconds 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
head -c 4000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
