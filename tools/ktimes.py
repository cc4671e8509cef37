"""Per-launch time / instructions from an `ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --csv` log."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
H = {h: j for j, h in enumerate(rows[i])}
d = {}
for r in rows[i + 1:]:
    d.setdefault((r[H["ID"]], r[H["Kernel Name"]]), {})[r[H["Metric Name"]]] = r[H["Metric Value"]]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for k, v in list(d.items())[:n]:
    print(f"{k[1][:48]:48s} {v.get('gpu__time_duration.sum'):>10s} {v.get('smsp__inst_executed.sum', ''):>12s}")
