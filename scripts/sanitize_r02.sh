# compute-sanitizer memcheck / racecheck / synccheck over the streamed int8 scan (with the bound
# epochs crossing the 32-bit wrap) and the tcgen05 pair scan + merge, small shapes.  Logs -> gpurun_out/san/.
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  MC_S8_EPOCH0=0xfffffffd timeout 600 compute-sanitizer --tool $tool --show-backtrace device \
      python scripts/profile_case.py c2 --iters 4 --entries 3000 > gpurun_out/san/${tool}_s8.log 2>&1
  echo "$tool s8 rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/san/${tool}_s8.log | tail -2 | tr '\n' ' ')"
  timeout 900 compute-sanitizer --tool $tool --show-backtrace device \
      python scripts/profile_case.py c3 --iters 1 --entries 4096 --batch 64 > gpurun_out/san/${tool}_tc.log 2>&1
  echo "$tool tc rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/san/${tool}_tc.log | tail -2 | tr '\n' ' ')"
done
