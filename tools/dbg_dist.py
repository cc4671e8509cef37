import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gdp_synth as synth
import paper_1310_0041_b200 as gdp
nz, ny, nx = 48, 128, 256
I0 = torch.from_numpy(synth.make_stack(nx, ny, nz, 53, "u8")).cuda()
for cyc in (1, 2):
    o = gdp.default_opts(max_vcycles=cyc, rel_tol=1e-30, stagnation=0)
    ctx = gdp.Ctx(0)
    a, ra = gdp.gdp_diffuse_z(ctx, I0, opts=o, check=False)
    lb = gdp.Ctx(0, loopback=2)
    b, rb = gdp.gdp_diffuse_z(lb, I0, opts=o, check=False)
    d = (a - b).abs().cpu().numpy()
    print("cycles", cyc, "max", d.max(), "per-plane max:", np.round(d.max(axis=(1, 2)) * 1e6, 2).tolist())
    print("  rows max (plane 0):", np.nonzero(d[0].max(axis=1) > 0)[0][:20].tolist(), "cols:", np.nonzero(d[0].max(axis=0) > 0)[0][:20].tolist())
    for opt in (0, 3):
        o2 = gdp.default_opts(max_vcycles=cyc, rel_tol=1e-30, stagnation=0, fused=opt)
        c2, _ = gdp.gdp_diffuse_z(lb, I0, opts=o2, check=False)
        print("  loopback fused", opt, "vs single fused3:", float((a - c2).abs().max()))
    ctx.close(); lb.close()
