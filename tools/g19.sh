python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "diffuse or screened or destripe or out_of_core or decode or constant" 2>&1 | tail -1
timeout 200 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$1.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_$1.json')); print(d['value'], d['ms_per_step'], {k: (v['launches'], v['ms']) for k, v in d['roofline']['kernels'].items() if k in ('util', 'coarse')})"
