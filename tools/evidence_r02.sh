# Round-2 evidence on one B200 (run under gpurun): smoke, GPU tests, benches (C4
# default line, C3, C5, table phi, FP32 engine, gradient, reference arm), the ncu
# launch list, ncu --set full of one steady-state stage launch (stage >= 1) of C4,
# C3 and C5, and the oracle timing on the host cores.
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
tag=${1:-r02}
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
TNRD_PARITY_REPORT=gpurun_out/parity_$tag.json timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; python tools/bench_line.py C4 < gpurun_out/bench_$tag.json
timeout 300 python bench.py --config 1 --steps 1000 --no-cpu-baseline > gpurun_out/bench_c1_$tag.json 2>/dev/null; python tools/bench_line.py C1 < gpurun_out/bench_c1_$tag.json
timeout 300 python bench.py --config 2 --steps 1000 --no-cpu-baseline > gpurun_out/bench_c2_$tag.json 2>/dev/null; python tools/bench_line.py C2 < gpurun_out/bench_c2_$tag.json
timeout 300 python bench.py --config 3 --steps 1000 --no-cpu-baseline > gpurun_out/bench_c3_$tag.json 2>/dev/null; python tools/bench_line.py C3 < gpurun_out/bench_c3_$tag.json
timeout 300 python bench.py --config 5 --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_$tag.json 2>/dev/null; python tools/bench_line.py C5 < gpurun_out/bench_c5_$tag.json
timeout 300 python bench.py --phi table --no-cpu-baseline > gpurun_out/bench_table_$tag.json 2>/dev/null; python tools/bench_line.py table < gpurun_out/bench_table_$tag.json
timeout 300 python bench.py --engine fp32 --steps 5 --no-cpu-baseline > gpurun_out/bench_fp32_$tag.json 2>/dev/null; python tools/bench_line.py fp32 < gpurun_out/bench_fp32_$tag.json
timeout 300 python bench.py --mode grad --steps 5 --warmup 3 > gpurun_out/bench_grad_$tag.json 2>/dev/null; python tools/bench_line.py grad < gpurun_out/bench_grad_$tag.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$tag.json 2>/dev/null; tail -c 300 gpurun_out/bench_ref_$tag.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_l_$tag.log 2>&1
for c in 4 3 5; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_stage_kernel --launch-skip 9 --launch-count 1 \
     -o gpurun_out/${tag}_c${c}_stage python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_c${c}_ncu.log 2>&1
  tail -1 gpurun_out/${tag}_c${c}_ncu.log
done
ncu -i gpurun_out/${tag}_c4_stage.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_c4_src.csv 2>/dev/null
# the NCCL halo exchange on hardware: launch list of the 1-rank self send/recv slab test
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/nccl_self_launches_$tag.csv \
   python -m pytest tests/test_gpu_parity.py -q -k "nccl_self_exchange and 2" > gpurun_out/nccl_self_$tag.log 2>&1; tail -1 gpurun_out/nccl_self_$tag.log
grep -c ncclDevKernel gpurun_out/nccl_self_launches_$tag.csv
[ -n "$ORACLE_TIMING" ] && timeout 1800 python tools/oracle_timing.py > gpurun_out/oracle_timing_$tag.json 2> gpurun_out/oracle_timing_$tag.err; tail -6 gpurun_out/oracle_timing_$tag.err
