python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 240 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or screened or destripe or slice" 2>&1 | tail -3
timeout 200 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$1.json 2>gpurun_out/bench_$1.err; echo bench rc=$?; python -c "
import json; d=json.load(open('gpurun_out/bench_$1.json')); print(d['value'], d['ms_per_step']); [print(k, v) for k, v in d['roofline']['kernels'].items()]"
FUSED=3 NCU_K="${NCU_K:-k_pass2d}" NCU_C=${NCU_C:-2} bash tools/gpu_round.sh $1 full > /dev/null 2>&1; python tools/ncu_summary.py gpurun_out/full_$1.ncu-rep | python -c "
import json,sys; d=json.load(sys.stdin)
for k in d: print(k['kernel'][:40], round(k['time_s']*1e6,1), 'inst', k['inst_executed'], 'warps', k['warps_active_pct'], 'issue', k['issue_active_pct'], 'rd', k['dram_read_B']/1e6, 'wr', k['dram_write_B']/1e6, 'GBps', round(k['dram_GBps']), k['top_stalls'])"
