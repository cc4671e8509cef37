python -c "import __graft_entry__ as g; g.build()" || exit 1
for b in 1 2 4 8; do GDP_HOST_BATCHES=$b timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_b$b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_b$b.json')); print('batches $b', d['value'], d['ms_per_step'], d['e2e']['value'])"; done
