"""Summarise ncu reports into profiles/ (per-kernel time, dram bytes, throughput, stalls)."""
import csv, json, subprocess, sys, collections

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        def f(k):
            try: return float(d[k].replace(",", ""))
            except Exception: return None
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): f(k) for k in hdr
              if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")}
        top = dict(sorted(((k, v) for k, v in st.items() if v), key=lambda kv: -kv[1])[:6])
        t = f("gpu__time_duration.sum")
        tu = units[hdr.index("gpu__time_duration.sum")]
        t_s = t * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(tu, 1e-9)
        sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
        rd = f("dram__bytes_read.sum") * sc.get(units[hdr.index("dram__bytes_read.sum")], 1)
        wr = f("dram__bytes_write.sum") * sc.get(units[hdr.index("dram__bytes_write.sum")], 1)
        scale = 1
        res.append({"kernel": d["Kernel Name"], "grid": d.get("launch__grid_size"), "time_s": t_s,
                    "dram_read_B": rd * scale, "dram_write_B": wr * scale,
                    "dram_GBps": (rd + wr) * scale / t_s / 1e9,
                    "inst_executed": f("smsp__inst_executed.sum"),
                    "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
                    "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                    "registers": f("launch__registers_per_thread"), "top_stalls": top,
                    "l2_hit_pct": f("lts__t_sector_hit_rate.pct"),
                    "dram_pct_peak": f("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
                    "sm_pct_peak": f("sm__throughput.avg.pct_of_peak_sustained_elapsed")})
    return res

if __name__ == "__main__":
    print(json.dumps(raw(sys.argv[1]), indent=1))
