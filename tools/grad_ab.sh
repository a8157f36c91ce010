for n in "$@"; do
  if [ "$n" = base ]; then unset TNRD_LIB_OVERRIDE; else export TNRD_LIB_OVERRIDE=build/exp/lib_$n.so; fi
  timeout 200 python bench.py --mode grad --steps 5 --warmup 3 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', round(d['ms_per_step'],3), round(d['value'],2))"
done
