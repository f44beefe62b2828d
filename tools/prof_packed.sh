# ncu of the single-string kernel (config e): packed vs RXG_NO_PACKED
mkdir -p gpurun_out/pk
python bench.py --config e --no-cpu --no-e2e --steps 2 --warmup 3 > gpurun_out/pk/plain.json 2>&1 || exit 1
for v in packed nopack; do
  if [ $v = nopack ]; then export RXG_NO_PACKED=1; fi
  ncu --set full --clock-control none --import-source on -k regex:k_chunk --launch-skip 3 -c 1 -o gpurun_out/pk/e_$v \
      python bench.py --config e --no-cpu --no-e2e --steps 2 --warmup 3 > gpurun_out/pk/ncu_$v.log 2>&1
  ncu -i gpurun_out/pk/e_$v.ncu-rep --page raw --csv > gpurun_out/pk/raw_$v.csv 2>/dev/null
  ncu -i gpurun_out/pk/e_$v.ncu-rep --page source --csv > gpurun_out/pk/src_$v.csv 2>/dev/null
done
