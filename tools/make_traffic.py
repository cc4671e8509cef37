"""profiles/ncu_full_summary.json: DRAM bytes per launch of the bench's kernel classes (finest
level), from an ncu --set full summary (tools/ncu_summary.py output).  The largest-traffic
instance of each template variant is its finest-level launch; a class averages the variants it
contains with equal weight (each runs once per V-cycle at the finest level)."""
import json, re, sys, collections

rows = json.load(open(sys.argv[1]))
best = {}
for r in rows:
    name = r["kernel"].split("(")[0]
    b = r["dram_read_B"] + r["dram_write_B"]
    if name not in best or b > best[name]["bytes"]:
        best[name] = {"bytes": b, "time_s": r["time_s"]}
classes = collections.defaultdict(list)
for name, v in best.items():
    m = re.search(r"k_march3d<(\d+), (\d+), (\d+), (\d+)>", name)
    if m:
        tail, prolong, zc = int(m.group(1)), int(m.group(2)), int(m.group(3))
        if zc:  # z-coarsened transfers only occur below the finest level
            continue
        classes["up3d@L0" if prolong else "down3d@L0"].append(v)
        continue
    m = re.search(r"k_m3v<(\d+), (\d+), (\d+)(?:, \d+)?>", name)
    if m:  # vertical-pack z-march: TAIL 1 restricts (down), PROLONG or TAIL 2 (norms) is the up pass
        tail, prolong, zc = int(m.group(1)), int(m.group(2)), int(m.group(3))
        if zc:
            continue
        classes["up3d@L0" if (prolong or tail == 2) else "down3d@L0"].append(v)
        continue
    m = re.search(r"k_pass2d<(\d+), (\d+)>", name)
    if m:
        classes["down2d@L0" if int(m.group(2)) else "up2d@L0"].append(v)
        continue
    m = re.search(r"k_rows2d<(\d+), (\d+)(?:, (\d+))?>", name)
    if m:
        if m.group(3) is not None and int(m.group(2)) and int(m.group(3)):
            continue  # down pass with the FMG prolongation: once per solve, not per V-cycle
        classes["down2d@L0" if int(m.group(2)) else "up2d@L0"].append(v)
        continue
    if "k_init" in name:
        classes["init@L0"].append(v)
out = {c: {"dram_bytes_per_launch": sum(x["bytes"] for x in vs) / len(vs),
           "ncu_time_s_per_launch": sum(x["time_s"] for x in vs) / len(vs), "variants": len(vs)}
       for c, vs in classes.items()}
out["_source"] = sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]
print(json.dumps(out, indent=1))
