#!/bin/bash
# One GPU session: tests, bench, launch list and ncu --set full of the top kernels.
# usage (via gpurun): bash tools/gpu_round.sh TAG [what...]   what in {tests,bench,launches,full}
TAG=${1:-r}; shift
WHAT=${@:-tests bench launches full}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { cat gpurun_out/build_$TAG.log; exit 1; }
for w in $WHAT; do
case $w in
tests) timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/tests_$TAG.log;;
bench) timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; cat gpurun_out/bench_$TAG.json | head -c 600; echo;;
launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$TAG.csv python tools/prof_step.py 1 > gpurun_out/launches_$TAG.log 2>&1; echo "launches rc=$?"; python tools/launch_summary.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt 2>&1; cat gpurun_out/launches_$TAG.txt;;
full) timeout 500 ncu --set full --clock-control none --import-source on --profile-from-start off -k "regex:${NCU_K:-k_}" --launch-skip ${NCU_SKIP:-0} -c ${NCU_C:-12} -f -o gpurun_out/full_$TAG python tools/prof_step.py 1 0 ${FUSED:-1} > gpurun_out/full_$TAG.log 2>&1; echo "full rc=$?"; python tools/ncu_summary.py gpurun_out/full_$TAG.ncu-rep > gpurun_out/full_$TAG.json 2>&1; head -c 3000 gpurun_out/full_$TAG.json;;
esac
done
