python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_3d or diffuse_z or destripe" 2>&1 | tail -15
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_s2b.json 2>gpurun_out/bench_s2b.err; echo bench rc=$?; cat gpurun_out/bench_s2b.json; tail -3 gpurun_out/bench_s2b.err
