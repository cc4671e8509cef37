"""Loopback z-slab partition vs single rank (fused / reference schedules), one V-cycle, max |diff|."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gdp_synth as synth
import paper_1310_0041_b200 as gdp
for shape in [(48, 128, 256), (40, 130, 250), (27, 96, 200), (64, 130, 75)]:
    nz, ny, nx = shape
    I0 = torch.from_numpy(synth.make_stack(nx, ny, nz, 53, "u8")).cuda()
    ctx = gdp.Ctx(0)
    lb = gdp.Ctx(0, loopback=2)
    res = {}
    for name, c, f in [("s0", ctx, 0), ("s3", ctx, 3), ("s1", ctx, 1), ("l0", lb, 0), ("l3", lb, 3)]:
        o = gdp.default_opts(max_vcycles=1, rel_tol=1e-30, stagnation=0, fused=f, fmg=0)
        res[name] = gdp.gdp_diffuse_z(c, I0, opts=o, check=False)[0].cpu().numpy()
    print(shape, {k: float(np.abs(res[k] - res["s0"]).max()) for k in res})
    ctx.close(); lb.close()
