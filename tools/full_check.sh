set -x
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
TNRD_PARITY_REPORT=gpurun_out/parity_tc9.json timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_tc9.json 2> gpurun_out/bench_tc9.err; tail -c 3000 gpurun_out/bench_tc9.json
timeout 300 python bench.py --engine fp32 --no-cpu-baseline > gpurun_out/bench_fp32_9.json 2>/dev/null; tail -c 300 gpurun_out/bench_fp32_9.json
timeout 300 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_9.json 2>/dev/null; tail -c 300 gpurun_out/bench_c3_9.json
timeout 300 python bench.py --config 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_9.json 2>/dev/null; tail -c 300 gpurun_out/bench_c5_9.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_tc9.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_l9.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_stage_kernel --launch-skip 8 --launch-count 1 -o gpurun_out/tc9_stage python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/tc9_ncu.log 2>&1; tail -1 gpurun_out/tc9_ncu.log
