# single-string packed layout: ring shapes (RXG_CHUNK_SHAPE: 0 default 16x1x128B, 1 the 32-byte ring, 5 12x2x128B) vs the row layout (RXG_NO_PACKED)
v() { python bench.py --config $1 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step']*1e3,1), 'us')"; }
for sh in 0 1 5; do
  RXG_CHUNK_SHAPE=$sh python -m pytest tests/test_layouts_fuzz.py -x -q -m gpu -k chunk_kernel 2>&1 | tail -1 | sed "s/^/shape $sh tests: /" | tee -a gpurun_out/pk.txt
done
for i in 1 2; do
  for c in e; do
    for sh in 0 1 5; do echo "$c shape$sh $(RXG_CHUNK_SHAPE=$sh v $c)" | tee -a gpurun_out/pk.txt; done
    echo "$c nopack $(RXG_NO_PACKED=1 v $c)" | tee -a gpurun_out/pk.txt
  done
done
