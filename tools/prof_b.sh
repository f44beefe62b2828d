mkdir -p gpurun_out/prof
python bench.py --config b --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof/bench_b.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/prof/launches_b.csv python bench.py --config b --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fixed -s 3 -c 1 -o gpurun_out/prof/full_b python bench.py --config b --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof/ncu_b.log 2>&1
