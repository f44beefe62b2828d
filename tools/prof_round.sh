set -x
mkdir -p gpurun_out/prof
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/prof/bench_c.json 2> gpurun_out/prof/bench_c.err
python bench.py --config d --steps 5 --warmup 3 --no-cpu > gpurun_out/prof/bench_d.json 2> gpurun_out/prof/bench_d.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/launches_c.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_lines_tma -s 3 -c 1 -o gpurun_out/prof/full_c python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof/ncu_c.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_lines_tma -s 3 -c 1 -o gpurun_out/prof/full_d python bench.py --config d --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof/ncu_d.log 2>&1
ls -la gpurun_out/prof
