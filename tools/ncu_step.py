"""Whole-step DRAM traffic: run under
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --print-units base --clock-control none
        --profile-from-start off --csv --log-file gpurun_out/step.csv python tools/prof_step.py 1 0 35
then  python tools/ncu_step.py gpurun_out/step.csv > profiles/ncu_step_r02.json
(bytes-weighted over all kernels of one config-1 destripe step; ncu serialises kernels with cold-ish
caches, so the kernel time is longer than the bench's)."""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
iid = hdr.index("ID")
per = {}
for r in rows[h + 1:]:
    if len(r) <= iv:
        continue
    d = per.setdefault(r[iid], {"kernel": r[ik]})
    d[r[im]] = float(r[iv].replace(",", ""))
rd = sum(d.get("dram__bytes_read.sum", 0.0) for d in per.values())
wr = sum(d.get("dram__bytes_write.sum", 0.0) for d in per.values())
ns = sum(d.get("gpu__time_duration.sum", 0.0) for d in per.values())
print(json.dumps({"dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr, "kernel_ms": ns / 1e6,
                  "dram_GBps": (rd + wr) / ns if ns else None, "launches": len(per),
                  "source": "ncu --metrics dram__bytes_*.sum,gpu__time_duration.sum of tools/prof_step.py 1 0 35"},
                 indent=1))
