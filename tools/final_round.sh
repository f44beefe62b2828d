# Round-end evidence: GPU tests, full-size parity, all benches (+ reference arm),
# the (c) launch list and one full ncu capture of its kernel.
mkdir -p gpurun_out/final gpurun_out/bench
python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; tail -1 gpurun_out/final/pytest_gpu.log
python tools/full_parity.py > gpurun_out/final/full_parity.log 2>&1; tail -1 gpurun_out/final/full_parity.log
bash tools/bench_all.sh > /dev/null 2>&1; ls gpurun_out/bench | wc -l
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_c.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_lines_tma -s 3 -c 1 -o gpurun_out/final/full_c python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_lines_tma -s 3 -c 1 -o gpurun_out/final/full_d python bench.py --config d --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_chunk_tma -s 3 -c 1 -o gpurun_out/final/full_e python bench.py --config e --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_fixed -s 3 -c 1 -o gpurun_out/final/full_b python bench.py --config b --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ls gpurun_out/final
