# C3 A/B/C... of several library builds on one box (LIBS under paper_2503_11972_b200/), ROUNDS rounds.
for r in $(seq ${ROUNDS:-2}); do
  for lib in $LIBS; do
    MODMCACHE_LIB=paper_2503_11972_b200/$lib timeout 300 python bench.py --steps 200 --warmup 5 --no-big --cpu-seconds 0.1 > gpurun_out/ab3.json 2> gpurun_out/ab3.err
    python -c "import json;d=json.loads(open('gpurun_out/ab3.json').read());c=d['c3'];print('$lib', 'C3 step %.2f us  check %.2f  frac %.3f  e2e %.0f/s' % (1e3*c['ms_per_step'], 1e3*c['profile']['step_ms'], c['roofline']['frac'], c['e2e']['value']))" || tail -3 gpurun_out/ab3.err
  done
done
