python -c "import __graft_entry__ as g; g.build()" || exit 1
python tools/prof_step.py 1 0 3 > /dev/null 2>&1 && timeout 300 ncu --set full --clock-control none --import-source on --profile-from-start off -k "regex:k_rows2d" -c 2 -f -o gpurun_out/full_$1 python tools/prof_step.py 1 0 3 > /dev/null 2>&1; python tools/ncu_summary.py gpurun_out/full_$1.ncu-rep | python -c "
import json,sys; d=json.load(sys.stdin)
for k in d: print(k['kernel'][:40], k['grid'], round(k['time_s']*1e6,1), 'inst', k['inst_executed'], 'warps', k['warps_active_pct'], 'issue', k['issue_active_pct'], 'GBps', round(k['dram_GBps']), 'regs', k['registers'], k['top_stalls'])"
