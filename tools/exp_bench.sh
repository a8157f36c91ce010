#!/bin/bash
# usage: exp_bench.sh name1 name2 ... (explibs/lib_NAME.so; "base" = product lib)
for n in "$@"; do
  if [ "$n" = base ]; then unset TNRD_LIB_OVERRIDE; else export TNRD_LIB_OVERRIDE=explibs/lib_$n.so; fi
  out=$(timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/tmp/exp_bench_err.txt)
  line=$(echo "$out" | grep '^{"metric"' | tail -1)
  if [ -z "$line" ]; then echo "$n FAILED: $(tail -3 /tmp/exp_bench_err.txt | tr '\n' ' ')"; continue; fi
  echo "$line" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', round(d['roofline']['mean_launch_ms'],3), 'ms', round(d['value'],1), 'MPix/s')"
done
