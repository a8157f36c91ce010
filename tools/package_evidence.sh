# Copy one evidence run (tools/evidence_r02.sh TAG, merged back under gpurun_out/) into profiles/r02_*.
#   bash tools/package_evidence.sh TAG
tag=${1:?tag}
G=gpurun_out; P=profiles
for pair in "bench_$tag:r02_bench" "bench_c1_$tag:r02_c1_bench" "bench_c2_$tag:r02_c2_bench" "bench_c3_$tag:r02_c3_bench" \
            "bench_c5_$tag:r02_c5_bench" "bench_table_$tag:r02_table_bench" "bench_fp32_$tag:r02_fp32_bench" \
            "bench_grad_$tag:r02_grad_bench" "bench_ref_$tag:r02_ref_bench"; do
  src=${pair%%:*}; dst=${pair##*:}; [ -s $G/$src.json ] && tail -1 $G/$src.json > $P/$dst.json
done
cp $G/parity_$tag.json $P/r02_parity_margins.json
cp $G/launches_$tag.csv $P/r02_launches.csv
cp $G/nccl_self_launches_$tag.csv $P/r02_nccl_self_launches.csv
for c in 4 3 5; do python tools/ncu_summary.py $G/${tag}_c${c}_stage.ncu-rep --json $P/r02_c${c}_stage_kernel_ncu.json > /dev/null 2>&1; done
python - <<'PY'
import json
t = json.load(open('profiles/traffic.json'))
for c in (4, 3, 5):
    d = json.load(open(f'profiles/r02_c{c}_stage_kernel_ncu.json'))['launches'][0]
    t[f'C{c}/tensor'] = d['dram_read_bytes'] + d['dram_write_bytes']
    print('ncu C%d' % c, d['duration_ms'], 'issue', d['issue_active_pct'], 'smem', d['smem_wavefront_pct'], 'fma', d['pipe_fma_cycles_pct'],
          'xu', d['pipe_xu_pct'], 'alu', d['pipe_alu_pct'], 'inst', d['inst_executed'], 'dram', t[f'C{c}/tensor'])
json.dump(t, open('profiles/traffic.json', 'w'), indent=1)
for n in ['r02_bench', 'r02_c1_bench', 'r02_c2_bench', 'r02_c3_bench', 'r02_c5_bench', 'r02_table_bench', 'r02_fp32_bench', 'r02_grad_bench', 'r02_ref_bench']:
    d = json.load(open(f'profiles/{n}.json'))
    r = d.get('roofline') or {}
    print(n, round(d['value'], 4), d.get('ms_per_step'), r.get('mean_launch_ms'), r.get('frac'), r.get('fp32_equivalent_frac'),
          (d.get('e2e') or {}).get('value'), (r.get('tensor') or {}).get('achieved'))
m = json.load(open('profiles/r02_parity_margins.json'))
print('parity max', max((v, k) for k, v in m.items() if isinstance(v, (int, float)) and 'dPSNR' not in k))
PY
