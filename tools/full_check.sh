# Final evidence on one B200 (run under gpurun): smoke, GPU tests, benches, launch
# list and one ncu --set full capture of the tensor-engine stage kernel.
set -x
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
tag=${1:-final}
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
TNRD_PARITY_REPORT=gpurun_out/parity_$tag.json timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -c 400 gpurun_out/bench_$tag.json
timeout 300 python bench.py --engine fp32 --no-cpu-baseline > gpurun_out/bench_fp32_$tag.json 2>/dev/null
timeout 300 python bench.py --phi table --no-cpu-baseline > gpurun_out/bench_table_$tag.json 2>/dev/null
timeout 300 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_c3_$tag.json 2>/dev/null
timeout 300 python bench.py --config 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_$tag.json 2>/dev/null
timeout 300 python bench.py --mode grad --steps 3 --warmup 3 > gpurun_out/bench_grad_$tag.json 2>/dev/null
timeout 300 python bench.py --mode grad --engine fp32 --steps 3 --warmup 3 > gpurun_out/bench_grad_fp32_$tag.json 2>/dev/null
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$tag.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_l_$tag.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_stage_kernel --launch-skip 9 --launch-count 1 -o gpurun_out/${tag}_stage python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_ncu.log 2>&1; tail -1 gpurun_out/${tag}_ncu.log
timeout 600 python tools/grad_margins.py > gpurun_out/grad_margins_$tag.json 2>/dev/null; tail -c 200 gpurun_out/grad_margins_$tag.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --mode grad --steps 1 --warmup 1 > gpurun_out/grad_launches_$tag.csv 2>/dev/null
