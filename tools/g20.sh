python -c "import __graft_entry__ as g; g.build()" || exit 1
python tools/prof_step.py 1 0 3 > /dev/null 2>&1 && timeout 400 ncu --set full --clock-control none --import-source on --profile-from-start off -k "regex:k_march3d" -c 2 -f -o gpurun_out/m3d_$1 python tools/prof_step.py 1 0 3 > /dev/null 2>&1; echo ncu rc=$?; ls -la gpurun_out/m3d_$1.ncu-rep
