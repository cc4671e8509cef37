python -c "import __graft_entry__ as g; g.build()" >/dev/null || exit 1
mkdir -p gpurun_out
timeout 300 python tools/prof_step.py 1 0 3 > gpurun_out/pz.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off --kernel-name-base mangled -k "regex:k_march3dILi0ELb1ELb1E" -c 4 -f -o gpurun_out/zc python tools/prof_step.py 1 0 3 > gpurun_out/zc_ncu.log 2>&1
echo ncu rc=$?
tail -3 gpurun_out/zc_ncu.log
ls -la gpurun_out/zc.ncu-rep
