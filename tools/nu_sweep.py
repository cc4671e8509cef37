"""Phase timings / V-cycle counts on config 1 for several (nu_pre, nu_post) per phase."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gdp_synth as synth
import paper_1310_0041_b200 as gdp
ctx = gdp.Ctx(0)
I0 = torch.from_numpy(synth.make_config(1)).cuda()
I1 = torch.empty(I0.shape, dtype=torch.float32, device="cuda")
I2 = torch.empty_like(I1)
for nu in [(2, 2), (1, 1), (2, 1), (1, 2), (3, 3)]:
    o = gdp.default_opts(nu_pre=nu[0], nu_post=nu[1], nu_pre_slices=nu[0], nu_post_slices=nu[1])
    res = []
    for rep in range(3):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        _, r1 = gdp.gdp_diffuse_z(ctx, I0, I1=I1, opts=o)
        e[1].record()
        _, r2 = gdp.gdp_screened_poisson_slices(ctx, I0, I1, I2=I2, alpha=0.01, opts=o)
        e[2].record()
        torch.cuda.synchronize()
        res.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), r1["vcycles"], r2["vcycles"], r1["rel_res"][-1], r2["rel_res"][-1]))
    print("nu", nu, "phase1 ms %.2f phase2 ms %.2f cycles %d %d rel %.2e %.2e" % min(res), flush=True)
