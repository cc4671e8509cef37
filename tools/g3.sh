python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_s2c.json 2>gpurun_out/bench_s2c.err; echo bench rc=$?; cat gpurun_out/bench_s2c.json; tail -3 gpurun_out/bench_s2c.err
FUSED=3 NCU_K="k_march3d" NCU_C=3 bash tools/gpu_round.sh s2c_m3d full
rm -f gpurun_out/*.ncu-rep
