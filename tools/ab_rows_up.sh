python -c "import __graft_entry__ as g; g.build()" || exit 1
for v in 0 1; do if [ $v = 1 ]; then export GDP_ROWS_UP=1; fi; timeout 200 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ru_$v.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/ru_$v.json')); print('rows_up=$v', d['value'], d['ms_per_step'], {k: (v['launches'], v['ms']) for k, v in d['roofline']['kernels'].items() if '2d' in k})"; done
GDP_ROWS_UP=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_2d or screened or destripe" 2>&1 | tail -1
