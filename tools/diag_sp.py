"""Phase-2 residual histories, fused vs reference schedule (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gdp_synth as synth
import paper_1310_0041_b200 as gdp
nz = int(sys.argv[1]) if len(sys.argv) > 1 else 16
ctx = gdp.Ctx(0)
I0 = torch.from_numpy(synth.make_config(1, nz=nz)).cuda()
I1, r1 = gdp.gdp_diffuse_z(ctx, I0)
for fused in (0, 1):
    o = gdp.default_opts(fused=fused)
    I2, r = gdp.gdp_screened_poisson_slices(ctx, I0, I1, alpha=0.01, opts=o)
    print("fused", fused, "cyc", r["vcycles"], " ".join("%.2e" % v for v in r["rel_res"]), "ms %.2f" % (r["seconds"] * 1e3))
    # fixed 4 cycles then recompute norms with the reference kernel
    o = gdp.default_opts(fused=fused, max_vcycles=4, rel_tol=1e-30, stagnation=0)
    I2, r = gdp.gdp_screened_poisson_slices(ctx, I0, I1, alpha=0.01, opts=o, check=False)
    o2 = gdp.default_opts(fused=0, max_vcycles=1, rel_tol=1e-30)
    print("   after 4 cycles reported", " ".join("%.2e" % v for v in r["rel_res"]))
    torch.save(I2.cpu(), f"/tmp/I2_{fused}.pt")
a, b = torch.load("/tmp/I2_0.pt"), torch.load("/tmp/I2_1.pt")
print("bitwise equal after 4 cycles:", torch.equal(a, b), (a - b).abs().max().item())
