python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "out_of_core or destripe" 2>&1 | tail -2
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_$1.json 2>gpurun_out/bench_$1.err; echo bench rc=$?; python -c "
import json; d=json.load(open('gpurun_out/bench_$1.json')); print(d['value'], d['ms_per_step'], d['e2e'])"
