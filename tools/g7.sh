python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 400 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 200 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$1.json 2>gpurun_out/bench_$1.err; echo bench rc=$?; python -c "
import json; d=json.load(open('gpurun_out/bench_$1.json')); print(d['value'], d['ms_per_step']); [print(k, v) for k, v in d['roofline']['kernels'].items()]"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$1.csv python tools/prof_step.py 1 0 3 > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/launches_$1.csv
