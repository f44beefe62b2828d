mkdir -p gpurun_out/prof
python bench.py --config e --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof/bench_e.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/prof/launches_e.csv python bench.py --config e --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_chunk_tma -s 4 -c 2 -o gpurun_out/prof/full_e python bench.py --config e --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof/ncu_e.log 2>&1
