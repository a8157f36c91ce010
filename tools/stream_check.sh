#!/bin/bash
# Streaming-engine development check on one B200 (run under gpurun): a quick parity
# subset, then C4 / C3 bench on the streaming and the per-tile engine.
#   bash tools/stream_check.sh TAG [full]
tag=${1:-dev}
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
if [ "$2" = full ]; then
  TNRD_PARITY_REPORT=gpurun_out/parity_$tag.json timeout 1800 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -6
else
  TNRD_PARITY_REPORT=gpurun_out/parity_$tag.json timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 \
    -k "full_config or engine_parity or r2_boundary or tile_edges or loopback or bitwise or ragged or c4_full or nccl_self" 2>&1 | tail -6
fi
for eng in stream tile; do
  if [ $eng = tile ]; then unset TNRD_STREAM; else export TNRD_STREAM=1; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${tag}_$eng.json 2> gpurun_out/bench_${tag}_$eng.err
  timeout 300 python bench.py --config 3 --steps 200 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/bench_${tag}_c3_$eng.json 2>> gpurun_out/bench_${tag}_$eng.err
  python - <<PY || tail -5 gpurun_out/bench_${tag}_$eng.err
import json
for c in ("", "_c3"):
    d = json.loads(open("gpurun_out/bench_${tag}" + c + "_$eng.json").read().strip().splitlines()[-1])
    print("$eng", c or "_c4", "MPix/s", round(d["value"], 1), "launch_ms", round(d["roofline"]["mean_launch_ms"], 3), "frac", round(d["roofline"]["frac"], 3), "clk", d["clocks"])
PY
done
unset TNRD_STREAM
