# End-to-end `rxvm match` on the GPU: the full config (c) file (1.02 GB,
# 10M lines) through paper_1108_3126_b200/rxgmatch, stdin to stdout.
set -e
python - <<'PY'
import sys; sys.path.insert(0, ".")
from paper_1108_3126_b200 import rx
rx.synth_input("c").tofile("/tmp/c.txt")
open("/tmp/c.pat", "w").write(rx.synth_pattern("c"))
PY
ls -la /tmp/c.txt
g++ -O2 -I/usr/local/cuda/include tools/cuda_init_probe.cpp -L/usr/local/cuda/lib64 -lcudart -o /tmp/cuda_init_probe && for i in 1 2 3; do /tmp/cuda_init_probe; done
P="$(cat /tmp/c.pat)"
./paper_1108_3126_b200/rxgmatch "$P" < /tmp/c.txt > /dev/null   # warm (page cache, driver)
RXGMATCH_TIMES=2 ./paper_1108_3126_b200/rxgmatch "$P" < /tmp/c.txt > /tmp/out.txt
for i in 1 2 3; do
  s=$(date +%s.%N); ./paper_1108_3126_b200/rxgmatch "$P" < /tmp/c.txt > /tmp/out.txt; e=$(date +%s.%N)
  python -c "print('rxgmatch wall %.3f s = %.2f GB/s' % ($e - $s, 1020819674 / ($e - $s) / 1e9))"
done
wc -l /tmp/out.txt
