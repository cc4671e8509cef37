import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
os.environ.setdefault("GDP_F3D_MIN", "0")
import numpy as np, torch
import gdp_synth as synth
import paper_1310_0041_b200 as gdp
ctx = gdp.Ctx(0)
I0 = synth.make_stack(65, 63, 9, 71, "f32")
for f in (0, 3, 35, 33, 34):
    out, rep = gdp.gdp_npr_filter(ctx, torch.from_numpy(I0).cuda(), alpha=0.01, lam=1.0, sigma=0.05, opts=gdp.default_opts(fused=f))
    print(f, rep["status"], rep["vcycles"], rep["rel_res"][:5], float(out.double().sum()))
