#!/bin/bash
# k-gradient kernel time per variant lib (build/exp/lib_NAME.so; "base" = product lib)
for n in "$@"; do
  if [ "$n" = base ]; then unset TNRD_LIB_OVERRIDE; else export TNRD_LIB_OVERRIDE=build/exp/lib_$n.so; fi
  t=$(timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"kgrad" -c 2 --csv python bench.py --mode grad --steps 1 --warmup 0 2>/dev/null | grep -o "\"[0-9.]*\"$" | tr -d '"' | tr '\n' ' ')
  echo "$n kgrad_ns: $t"
done
