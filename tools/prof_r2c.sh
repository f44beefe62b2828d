# Final round-2 evidence: default bench line, its launch list, one ncu --set
# full capture each of the headline kernel and of the kernels changed late in
# the round. Output: gpurun_out/r2_end/ (summaries; .ncu-rep stay in /tmp).
set -x
O=gpurun_out/r2_end
mkdir -p $O
python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-sub --bitset-subs "" --k1-subs "" > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c_results.csv python tools/res_lines.py c > /dev/null 2>&1
cap() {  # name kernel-regex skip command...
  n=$1; k=$2; s=$3; shift 3
  ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o /tmp/$n "$@" > $O/ncu_$n.log 2>&1
  python tools/ncu_summary.py /tmp/$n.ncu-rep > $O/ncu_full_$n.txt 2>&1
  python tools/ncu_source.py /tmp/$n.ncu-rep 25 > $O/ncu_source_$n.txt 2>&1
}
cap c k_lines_tma 3 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-sub --bitset-subs "" --k1-subs ""
cap b k_fixed_tma 3 python bench.py --config b --steps 1 --warmup 3 --no-cpu --no-e2e --no-sub --bitset-subs "" --k1-subs ""
cap e k_chunk_tma 3 python bench.py --config e --steps 1 --warmup 3 --no-cpu --no-e2e --no-sub --bitset-subs "" --k1-subs ""
cap c_results k_lines_tma 13 python tools/res_lines.py c
cap c_scatter k_lt_scatter 3 python tools/res_lines.py c
python tools/res_lines.py c d > $O/res_lines_cd.txt 2>&1
python tools/cliff.py > $O/cliff.txt 2>&1
python tools/copy_threads.py 8 16 > $O/copy_threads.txt 2>&1
bash tools/rxgmatch_e2e.sh > $O/rxgmatch_e2e.txt 2>&1
ls -la $O
