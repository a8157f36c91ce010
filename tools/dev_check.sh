# Development loop on the GPU box: smoke, GPU tests (optionally a subset), short bench.
#   bash tools/dev_check.sh TAG [pytest-args...]
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
tag=${1:-dev}; shift
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
TNRD_PARITY_REPORT=gpurun_out/parity_$tag.json timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 "$@" 2>&1 | tail -15 > gpurun_out/tests_$tag.log; tail -6 gpurun_out/tests_$tag.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_$tag.json').read().strip().splitlines()[-1])
print('BENCH', d['value'], 'MPix/s', 'launch_ms', d['roofline']['mean_launch_ms'], 'frac', d['roofline']['frac'])" || tail -5 gpurun_out/bench_$tag.err
timeout 300 python bench.py --config 3 --steps 1000 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_$tag.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/bench_c3_$tag.json').read().strip().splitlines()[-1])
print('C3', d['value'], 'MPix/s', 'launch_ms', d['roofline']['mean_launch_ms'], 'frac', d['roofline']['frac'])"
