#!/bin/bash
# A/B on the GPU: bench value of the working tree vs a git ref (stash-free: the ref is built in /tmp)
# usage: bash tools/ab_bench.sh [REF]   (REF default HEAD)
REF=${1:-HEAD}
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('new', d['value'], d['ms_per_step'], d['vcycles']['phase1'], d['vcycles']['phase2'])"; done
