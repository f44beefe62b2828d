mkdir -p gpurun_out/prof
python -m pytest tests/test_gpu_stress.py -x -q -k "fixed" 2>&1 | tail -1
for i in 1 2; do python bench.py --config b --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])"; done
ncu --set full --clock-control none --import-source on -k regex:k_fixed -s 3 -c 1 -o gpurun_out/prof/full_b3 python bench.py --config b --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof/ncu_b3.log 2>&1
