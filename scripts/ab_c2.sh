# A/B of two library builds on the same box: C2 bench line, alternating, 3 rounds each.
#   A = paper_2503_11972_b200/libmodmcache.so, B = $B (default paper_2503_11972_b200/libB.so)
B=${B:-paper_2503_11972_b200/libB.so}
for r in 1 2; do
  for lib in paper_2503_11972_b200/libmodmcache.so $B; do
    MODMCACHE_LIB=$lib timeout 300 python bench.py --steps ${STEPS:-3000} --warmup 5 --no-c3 --cpu-seconds 0.1 > gpurun_out/ab.json 2> gpurun_out/ab.err
    python -c "import json;d=json.loads(open('gpurun_out/ab.json').read());print('$lib'.split('/')[-1], 'step %.2f us  e2e %.0f/s  check %.2f us' % (1e3*d['ms_per_step'], d['e2e']['value'], 1e3*d['profile']['step_ms']))" || tail -3 gpurun_out/ab.err
  done
done
