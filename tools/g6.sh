python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python tools/nu_sweep.py 2>&1 | tail -8
timeout 300 ncu --set full --clock-control none --profile-from-start off -k "regex:k_coarse_fd|k_norms|k_rhs" -c 4 -f -o gpurun_out/full_s2h python tools/prof_step.py 1 0 3 > /dev/null 2>&1; python tools/ncu_summary.py gpurun_out/full_s2h.ncu-rep | python -c "
import json,sys; d=json.load(sys.stdin)
for k in d: print(k['kernel'][:40], k['grid'], round(k['time_s']*1e6,1), 'inst', k['inst_executed'], 'warps', k['warps_active_pct'], 'issue', k['issue_active_pct'], 'GBps', round(k['dram_GBps']), k['top_stalls'])"
