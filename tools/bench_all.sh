# All configs through bench.py (defaults: CPU baseline + e2e), then the reference arm for (c).
# QUICK=1: no CPU legs, no reference arm.
mkdir -p gpurun_out/bench
extra=""
[ -n "$QUICK" ] && extra="--no-cpu"
for c in c d b e a; do
  python bench.py --config $c $extra > gpurun_out/bench/bench_$c.json 2> gpurun_out/bench/bench_$c.err
  tail -1 gpurun_out/bench/bench_$c.json | cut -c1-200
done
if [ -z "$QUICK" ]; then
  python bench.py --impl reference > gpurun_out/bench/ref_c.json 2> gpurun_out/bench/ref_c.err
  tail -1 gpurun_out/bench/ref_c.json | cut -c1-200
fi
