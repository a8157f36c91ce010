# ncu --set full of one steady-state C4 stage launch per variant lib (explibs/lib_NAME.so,
# "base" = product).  usage: ncu_ab.sh TAG name1 name2 ...
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
tag=$1; shift
for n in "$@"; do
  if [ "$n" = base ]; then unset TNRD_LIB_OVERRIDE; else export TNRD_LIB_OVERRIDE=explibs/lib_$n.so; fi
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_stage_kernel --launch-skip 9 --launch-count 1 \
     -o gpurun_out/${tag}_$n python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_${n}_ncu.log 2>&1
  tail -1 gpurun_out/${tag}_${n}_ncu.log
  ncu -i gpurun_out/${tag}_$n.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_${n}_src.csv 2>/dev/null
done
