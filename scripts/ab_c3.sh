# A/B of two library builds on one box: the bench's C3 line (and C2, which runs first), 2 rounds.
B=${B:-paper_2503_11972_b200/libB.so}
for r in 1 2; do
  for lib in paper_2503_11972_b200/libmodmcache.so $B; do
    MODMCACHE_LIB=$lib timeout 300 python bench.py --steps 40 --warmup 5 --no-big --cpu-seconds 0.1 > gpurun_out/ab3.json 2> gpurun_out/ab3.err
    python -c "import json;d=json.loads(open('gpurun_out/ab3.json').read());c=d['c3'];print('$lib'.split('/')[-1], 'C3 step %.2f us  check %.2f  e2e %.0f/s | C2 %.2f us' % (1e3*c['ms_per_step'], 1e3*c['profile']['step_ms'], c['e2e']['value'], 1e3*d['ms_per_step']))" || tail -3 gpurun_out/ab3.err
  done
done
