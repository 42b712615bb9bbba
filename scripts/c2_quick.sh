# C2 iteration loop on the GPU box: phase stamps (rotated caches), then the bench's C2 line only.
MC_GEMV_TIMING=1 timeout 120 python scripts/profile_case.py c2 --iters 8 --rotate 4 > gpurun_out/phases.log 2>&1
grep -A1 "^stream8" gpurun_out/phases.log | tail -2; grep median gpurun_out/phases.log | tail -1
timeout 300 python bench.py --steps ${STEPS:-2000} --warmup 5 --no-c3 --cpu-seconds 0.5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_c2.json").read())
print("C2 value %.0f/s  ms_per_step %.2f us  frac %.3f  e2e %.0f/s  cpu %.0f/s  clocks %s" % (
    d["value"], 1e3 * d["ms_per_step"], d["roofline"]["frac"], d["e2e"]["value"], d["cpu_baseline"]["value"], d["clocks"]))
PY
tail -3 gpurun_out/bench_c2.err
