#!/bin/bash
# Development loop on the GPU box: parity tests, a short bench, optionally one
# ncu --set full capture of a stage launch.  Usage (inside gpurun):
#   bash tools/gpu_check.sh TAG [tests] [ncu]
tag=${1:-dev}; shift
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
for what in "$@"; do
  case $what in
    tests) TNRD_PARITY_REPORT=gpurun_out/parity_$tag.json timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 ;;
  esac
done
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_$tag.json').read().strip().splitlines()[-1])
print('BENCH', d['value'], 'MPix/s', 'launch_ms', d['roofline']['mean_launch_ms'], 'frac', d['roofline']['frac'])" || tail -5 gpurun_out/bench_$tag.err
for what in "$@"; do
  case $what in
    ncu) timeout 600 ncu --set full --import-source on --clock-control none -k regex:stage_kernel --launch-skip 9 --launch-count 1 \
           -o gpurun_out/${tag}_stage python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_ncu.log 2>&1; tail -1 gpurun_out/${tag}_ncu.log ;;
  esac
done
