#!/bin/bash
# Round profile: bench JSON, launch list of the bench command, ncu --set full of the finest-level
# kernels -> gpurun_out/*_$TAG.*   (copy the summaries to profiles/)
TAG=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail gpurun_out/build_$TAG.log; exit 1; }
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > /dev/null 2>&1
echo "launches rc=$?"
python tools/launch_summary.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt 2>&1
timeout 300 python tools/prof_step.py 1 0 35 > gpurun_out/plain2_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k "regex:k_m3v|k_march3d|k_init" -c 130 -f -o gpurun_out/prof3d_$TAG python tools/prof_step.py 1 0 35 > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k "regex:k_pass2d|k_rows2d" -c 30 -f -o gpurun_out/prof2d_$TAG python tools/prof_step.py 1 0 35 > /dev/null 2>&1
echo "ncu rc=$?"
python - <<PY
import json, subprocess
rows = []
for r in ("prof3d_$TAG", "prof2d_$TAG"):
    out = subprocess.run(["python", "tools/ncu_summary.py", f"gpurun_out/{r}.ncu-rep"], capture_output=True, text=True).stdout
    try: rows += json.loads(out)
    except Exception as e: print("summary failed", r, e)
json.dump(rows, open("gpurun_out/ncu_full_$TAG.json", "w"), indent=1)
PY
python tools/make_traffic.py gpurun_out/ncu_full_$TAG.json "ncu --set full of tools/prof_step.py 1 0 35 (profiles/ncu_full_$TAG.json)" > gpurun_out/ncu_full_summary.json
rm -f gpurun_out/prof3d_$TAG.ncu-rep gpurun_out/prof2d_$TAG.ncu-rep; ls -la gpurun_out/*.ncu-rep
du -sh gpurun_out; free -g | head -2; nproc; df -h /dev/shm /tmp | tail -2
