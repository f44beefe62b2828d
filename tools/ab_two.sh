# A/B of the working-tree library against ab/librxg_$1.so on configs $2.. (bench.py device time)
old=$PWD/ab/librxg_$1.so; shift
for c in "$@"; do
  for i in 1 2; do
    n=$(python bench.py --config $c --steps 20 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],1))")
    o=$(RXG_LIB=$old python bench.py --config $c --steps 20 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],1))")
    echo "$c new $n old $o"
  done
done
