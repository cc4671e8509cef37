import os, sys
sys.path.insert(0, os.getcwd())
import torch
import gdp_synth as synth
import paper_1310_0041_b200 as gdp
ctx = gdp.Ctx(0)
I0 = torch.from_numpy(synth.make_config(1)).cuda()
I1 = torch.empty(I0.shape, dtype=torch.float32, device="cuda"); I2 = torch.empty_like(I1)
for nu in ["default"]:  # (GDP_FMG_NU overrides were removed; kept for the record)
    os.environ["GDP_FMG_NU"] = nu
    for ph in (1, 2):
        best = None
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = gdp.gdp_diffuse_z(ctx, I0, I1=I1, check=False)[1] if ph == 1 else gdp.gdp_screened_poisson_slices(ctx, I0, I1, I2=I2, alpha=0.01, check=False)[1]
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1); best = ms if best is None else min(best, ms)
        print("fmg nu", nu, "phase", ph, round(best, 3), r["vcycles"], ["%.2e" % v for v in r["rel_res"][:r["vcycles"] + 1]], flush=True)
