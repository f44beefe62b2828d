# A/B of chunk-engine builds on config (e) (ab/librxg_*.so from variant builds): device ms per step.
for lib in "" $(ls ab/librxg_*.so 2>/dev/null); do
  for i in 1 2; do
    RXG_LIB=$lib python bench.py --config e --no-sub --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('${lib:-base}', round(d['ms_per_step']*1e3,2), 'us', round(d['value']), 'GB/s')"
  done
done
