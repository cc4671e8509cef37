#!/bin/bash
# A/B of prebuilt variants (variants/libgdp_X.so; the in-tree library is A) on the TMA-staged 3D
# sweep: bench ms/step twice, then ncu DRAM bytes + time of the k_m3v launches of one step
# -> gpurun_out/abtma_<X>.csv and a per-variant summary line per kernel template
# usage (via gpurun): bash tools/ab_tma.sh X ...
mkdir -p gpurun_out
cp paper_1310_0041_b200/libgdp.so /tmp/libgdp_A.so
run() {
  for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-alpha-sweep 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$1', round(d['ms_per_step'],3), d['phase_ms_median'], d['vcycles']['phase1'], d['vcycles']['phase2'])"; done
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off -k regex:k_m3v --csv --log-file gpurun_out/abtma_$1.csv python tools/prof_step.py 1 > /dev/null 2>&1
  python - <<PY
import csv, collections
rows = list(csv.reader(open("gpurun_out/abtma_$1.csv")))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
H = {h: j for j, h in enumerate(rows[i])}
acc = collections.defaultdict(lambda: collections.defaultdict(float)); best = {}
per = collections.defaultdict(dict)
for r in rows[i + 1:]:
    if len(r) < len(H): continue
    per[(r[H["ID"]], r[H["Kernel Name"]].split("(")[0])][r[H["Metric Name"]]] = (float(r[H["Metric Value"]].replace(",", "")), r[H["Metric Unit"]])
for (id_, k), m in per.items():
    t, tu = m["gpu__time_duration.sum"]; t *= {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(tu, 1e-6)
    rd, ru = m["dram__bytes_read.sum"]; rd *= {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(ru, 1e-9)
    if k not in best or rd > best[k][1]: best[k] = (t, rd)
for k, (t, rd) in sorted(best.items()): print("$1", k, "finest launch: %.3f ms, DRAM read %.3f GB" % (t, rd))
PY
}
run A
for v in "$@"; do
  cp variants/libgdp_$v.so paper_1310_0041_b200/libgdp.so && touch paper_1310_0041_b200/libgdp.so && run $v
done
cp /tmp/libgdp_A.so paper_1310_0041_b200/libgdp.so
