"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel name."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0][:60]
    v = float(r[vi].replace(",", ""))
    unit = hdr[vi]
    agg[name][0] += 1
    agg[name][1] += v
    tot += v
print(f"{'kernel':60s} {'launches':>8s} {'total':>12s} {'share':>6s} {'avg':>10s}")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:60s} {n:8d} {t:12.0f} {100*t/tot:5.1f}% {t/n:10.0f}")
print(f"total {tot:.0f} (ns) over {sum(n for n,_ in agg.values())} launches")
