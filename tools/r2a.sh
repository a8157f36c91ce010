export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
TNRD_PARITY_REPORT=gpurun_out/parity_r2a.json timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1200 2>&1 | tail -15 > gpurun_out/tests_r2a.log; tail -5 gpurun_out/tests_r2a.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; tail -c 600 gpurun_out/bench_r2a.json
