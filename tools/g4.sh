python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 240 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_3d or diffuse_z or destripe" 2>&1 | tail -3
timeout 200 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_s2e.json 2>gpurun_out/bench_s2e.err; echo bench rc=$?; python -c "
import json; d=json.load(open('gpurun_out/bench_s2e.json')); print(d['value'], d['ms_per_step']); [print(k, v) for k, v in d['roofline']['kernels'].items()]"
FUSED=3 NCU_K="k_march3d" NCU_C=3 bash tools/gpu_round.sh s2e_m3d full > /dev/null 2>&1; python tools/ncu_summary.py gpurun_out/full_s2e_m3d.ncu-rep | python -c "
import json,sys; d=json.load(sys.stdin)
for k in d: print(k['kernel'][:40], k['time_s']*1e6, 'inst', k['inst_executed'], 'warps', k['warps_active_pct'], 'issue', k['issue_active_pct'], k['top_stalls'])"
