#!/bin/bash
# Quick GPU check (via gpurun): build, a pytest -k selection, the bench line.
#   bash tools/gpu_check.sh TAG "pytest -k expression"
TAG=${1:-chk}; SEL=${2:-}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
if [ -n "$SEL" ]; then timeout 600 python -m pytest tests -x -q -m gpu -k "$SEL" 2>&1 | tail -3; fi
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.json 2>gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print(d['value'], d['ms_per_step'])
for k, v in d['roofline']['kernels'].items(): print(' ', k, v)"
