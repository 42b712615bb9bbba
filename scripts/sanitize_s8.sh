set -x
timeout 300 compute-sanitizer --tool memcheck --show-backtrace device python scripts/profile_case.py c2 --iters 1 --entries 3000 > gpurun_out/sanitize.log 2>&1; echo rc=$?
head -60 gpurun_out/sanitize.log
