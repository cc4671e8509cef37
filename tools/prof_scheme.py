"""One Hybrid / Linear phase-1 solve of config 1 under cudaProfilerStart/Stop (ncu --profile-from-start off)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gdp_synth as synth
import paper_1310_0041_b200 as gdp

scheme = sys.argv[1] if len(sys.argv) > 1 else "hybrid"
ctx = gdp.Ctx(0)
I0 = torch.from_numpy(synth.make_config(1)).cuda()
o = gdp.default_opts(scheme=scheme)
gdp.gdp_diffuse_z(ctx, I0, opts=o)
torch.cuda.synchronize()
torch.cuda.profiler.start()
I1, r = gdp.gdp_diffuse_z(ctx, I0, opts=o)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ms", r["seconds"] * 1e3, "cycles", r["vcycles"])
