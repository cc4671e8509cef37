"""One warm destripe step under cudaProfilerStart/Stop (for ncu --profile-from-start off)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gdp_synth as synth
import paper_1310_0041_b200 as gdp

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
nz = (int(sys.argv[2]) or None) if len(sys.argv) > 2 else None
fused = int(sys.argv[3]) if len(sys.argv) > 3 else None  # None: the library default
ctx = gdp.Ctx(0)
I0 = torch.from_numpy(synth.make_config(cfg, nz=nz)).cuda()
o = gdp.default_opts() if fused is None else gdp.default_opts(fused=fused)
for _ in range(2):
    gdp.gdp_destripe(ctx, I0, opts=o)
torch.cuda.synchronize()
torch.cuda.profiler.start()
I1, I2, r1, r2 = gdp.gdp_destripe(ctx, I0, opts=o)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("dev ms", r1["seconds"] * 1e3, r2["seconds"] * 1e3, "cycles", r1["vcycles"], r2["vcycles"])
