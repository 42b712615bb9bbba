# A/B/C... of several library builds on the same box: C2 bench line, alternating, $ROUNDS rounds each.
#   LIBS="a.so b.so ..." (paths under paper_2503_11972_b200/)
for r in $(seq ${ROUNDS:-2}); do
  for lib in $LIBS; do
    MODMCACHE_LIB=paper_2503_11972_b200/$lib timeout 300 python bench.py --steps ${STEPS:-3000} --warmup 5 --no-c3 --cpu-seconds 0.1 > gpurun_out/ab.json 2> gpurun_out/ab.err
    python -c "import json;d=json.loads(open('gpurun_out/ab.json').read());print('$lib', 'step %.2f us  e2e %.0f/s  seq %.0f/s  e2e lat %.1f us' % (1e3*d['ms_per_step'], d['e2e']['value'], d['e2e']['sequential']['value'], d['e2e']['latency_us']))" || tail -3 gpurun_out/ab.err
  done
done
