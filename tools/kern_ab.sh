#!/bin/bash
# usage: kern_ab.sh REGEX name1 name2 ... : per-launch ns of kernels matching REGEX in the
# gradient bench, per variant lib (explibs/lib_NAME.so; "base" = product lib)
re=$1; shift
for n in "$@"; do
  if [ "$n" = base ]; then unset TNRD_LIB_OVERRIDE; else export TNRD_LIB_OVERRIDE=explibs/lib_$n.so; fi
  t=$(timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$re" -c 2 --csv python bench.py --mode grad --steps 1 --warmup 0 2>/dev/null | grep -o "\"[0-9.]*\"$" | tr -d '"' | tr '\n' ' ')
  echo "$n $re ns: $t"
done
