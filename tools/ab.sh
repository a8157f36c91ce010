#!/bin/bash
# A/B of experiment libs: bench C4 (and C3 with C3=1) per variant; PARITY=name runs a parity subset on that variant.
#   bash tools/ab.sh name1 name2 ...     (explibs/lib_NAME.so; "base" = product lib)
mkdir -p gpurun_out
for n in "$@"; do
  if [ "$n" = base ]; then unset TNRD_LIB_OVERRIDE; else export TNRD_LIB_OVERRIDE=explibs/lib_$n.so; fi
  out=$(timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/tmp/ab_err.txt)
  line=$(echo "$out" | grep '^{"metric"' | tail -1)
  if [ -z "$line" ]; then echo "$n FAILED: $(tail -3 /tmp/ab_err.txt | tr '\n' ' ')"; continue; fi
  echo "$line" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n C4', round(d['roofline']['mean_launch_ms'],3), 'ms', round(d['value'],1), 'MPix/s')"
  if [ -n "$C3" ]; then
    timeout 300 python bench.py --config 3 --steps 600 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{"metric"' | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n C3', round(d['roofline']['mean_launch_ms']*1e3,2), 'us', round(d['value'],1), 'MPix/s')"
  fi
  if [ "$PARITY" = "$n" ] || [ "$PARITY" = all ]; then
    timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 600 -k "full_config_parity or bitwise_determinism or tile_edges or phi_micro or other_rbf or stress or ragged or engine_parity or c4_full_batch" 2>&1 | tail -3
  fi
done
