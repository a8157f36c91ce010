# Round-2 state check on one B200: smoke, full GPU suite, default bench, C3 bench.
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
tag=${1:-r2b}
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
TNRD_PARITY_REPORT=gpurun_out/parity_$tag.json timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 2>&1 | tail -15 > gpurun_out/tests_$tag.log; tail -5 gpurun_out/tests_$tag.log
timeout 300 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -c 1500 gpurun_out/bench_$tag.json
timeout 300 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_c3_$tag.json 2>/dev/null; tail -c 300 gpurun_out/bench_c3_$tag.json
