"""Per-phase smoothing (nu_pre, nu_post) with the FMG start on config 1: time, cycles, rel-res."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gdp_synth as synth
import paper_1310_0041_b200 as gdp
ctx = gdp.Ctx(0)
I0 = torch.from_numpy(synth.make_config(1)).cuda()
I1 = torch.empty(I0.shape, dtype=torch.float32, device="cuda"); I2 = torch.empty_like(I1)
def run(fn):
    best = None
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = fn(); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1); best = (ms, r) if best is None or ms < best[0] else best
    return best
for nu in [(2, 2), (2, 1), (1, 2), (1, 1), (3, 1)]:
    o = gdp.default_opts(nu_pre=nu[0], nu_post=nu[1])
    ms, (_, r) = run(lambda: gdp.gdp_diffuse_z(ctx, I0, I1=I1, opts=o, check=False))
    print(f"phase1 nu={nu}: {ms:.2f} ms cycles {r['vcycles']} rel {r['rel_res'][-1] if False else r['rel_res'][r['vcycles']]:.2e}", flush=True)
gdp.gdp_diffuse_z(ctx, I0, I1=I1)
for nu in [(1, 2), (1, 1), (2, 1), (2, 2)]:
    o = gdp.default_opts(nu_pre_slices=nu[0], nu_post_slices=nu[1])
    ms, (_, r) = run(lambda: gdp.gdp_screened_poisson_slices(ctx, I0, I1, I2=I2, alpha=0.01, opts=o, check=False))
    print(f"phase2 nu={nu}: {ms:.2f} ms cycles {r['vcycles']} rel {r['rel_res'][r['vcycles']]:.2e}", flush=True)
