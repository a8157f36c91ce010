#!/bin/bash
# per-role timers of the streaming kernel (explibs/lib_NAME.so built with TNRD_SX_PROF):
# prints the per-CTA average of each timer for the last stage launch of a C4 step
for n in "$@"; do
  TNRD_LIB_OVERRIDE=explibs/lib_$n.so timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 >/dev/null | grep SXPROF | tail -2 | sed "s/^/$n /"
done
