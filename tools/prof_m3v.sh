# ncu --set full of the finest-level k_m3v launches of one destripe step (fused 35) -> gpurun_out/m3v_*
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k "regex:k_m3v" --launch-skip ${1:-8} -c ${2:-3} -f -o gpurun_out/m3v python tools/prof_step.py 1 0 35 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/m3v.ncu-rep > gpurun_out/m3v_summary.json
for i in $(seq 0 $((${2:-3} - 1))); do
  ncu -i gpurun_out/m3v.ncu-rep --page source --csv --launch-skip $i --launch-count 1 > gpurun_out/m3v_src$i.csv 2>&1
done
ncu -i gpurun_out/m3v.ncu-rep --page details --csv > gpurun_out/m3v_details.csv 2>&1
rm -f gpurun_out/m3v.ncu-rep
