# C3 step timing: graph replay with and without per-launch events, and eager launches
python bench.py --config 3 --steps 1000 --no-cpu-baseline --no-e2e 2>/dev/null | python tools/bench_line.py graph+events
python bench.py --config 3 --steps 1000 --no-cpu-baseline --no-e2e --no-launch-events 2>/dev/null | python tools/bench_line.py graph
TNRD_GRAPH=0 python bench.py --config 3 --steps 1000 --no-cpu-baseline --no-e2e --no-launch-events 2>/dev/null | python tools/bench_line.py eager
