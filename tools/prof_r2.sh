# Round-2 evidence on one GPU box: default bench line, its ncu launch list,
# and one ncu --set full capture per kernel of interest, summarised with
# tools/ncu_summary.py (the .ncu-rep files stay on the box). Output: gpurun_out/r2/.
set -x
O=gpurun_out/r2
mkdir -p $O
python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-sub --bitset-subs "" --k1-subs "" > /dev/null 2>&1
cap() {  # name kernel-regex skip command...
  n=$1; k=$2; s=$3; shift 3
  ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o /tmp/$n "$@" > $O/ncu_$n.log 2>&1
  python tools/ncu_summary.py /tmp/$n.ncu-rep > $O/ncu_full_$n.txt 2>&1
  python tools/ncu_source.py /tmp/$n.ncu-rep 25 > $O/ncu_source_$n.txt 2>&1
}
cap c k_lines_tma 3 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-sub --bitset-subs "" --k1-subs ""
cap d k_lines_tma 3 python bench.py --config d --steps 1 --warmup 3 --no-cpu --no-e2e --no-sub --bitset-subs "" --k1-subs ""
cap c_bitset k_bits_tma 1 python tools/prof_bits.py c
cap d_bitset k_bits_tma 1 python tools/prof_bits.py d
cap e_k1 k_pernode 1 python tools/k1_e.py e
cap c_results k_lines_tma 13 python tools/res_lines.py c
ls -la $O
