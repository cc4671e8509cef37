"""Dynamic SASS opcode mix from `ncu --page source --csv` (per-instruction executed counts)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "Address"][0]
H = {h: j for j, h in enumerate(rows[i])}
mix = collections.Counter(); tot = 0
for r in rows[i + 1:]:
    if len(r) < len(H): continue
    try: n = float(r[H["Instructions Executed"]] or 0)
    except ValueError: continue
    src = r[H["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"): op = src.split()[1]
    mix[op.split(".")[0]] += n; tot += n
print("total", tot)
for op, n in mix.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{op:10s} {n:12.0f} {100*n/tot:5.1f}%")
