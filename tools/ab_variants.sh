#!/bin/bash
# A/B of prebuilt library variants on the GPU (no rebuild on the box): the in-tree libgdp.so is A,
# each variants/libgdp_X.so is swapped in turn.  Per variant: two bench lines (device ms/step,
# cycles) and the launch list of one step -> gpurun_out/ab_<X>.{txt,csv}
# usage (via gpurun): bash tools/ab_variants.sh [X ...]
mkdir -p gpurun_out
cp paper_1310_0041_b200/libgdp.so /tmp/libgdp_A.so
run() {
  for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$1', round(d['ms_per_step'],3), d['phase_ms_median'], d['vcycles']['phase1'], d['vcycles']['phase2'])"; done
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/ab_$1.csv python tools/prof_step.py 1 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/ab_$1.csv > gpurun_out/ab_$1.txt 2>&1
}
run A
for v in "$@"; do
  cp variants/libgdp_$v.so paper_1310_0041_b200/libgdp.so && touch paper_1310_0041_b200/libgdp.so && run $v
done
cp /tmp/libgdp_A.so paper_1310_0041_b200/libgdp.so
