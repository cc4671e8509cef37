"""FMG start vs plain start on config 1 (and config 2): per-phase time, cycle counts, rel-res
histories, and the difference of the converged answers."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gdp_synth as synth
import paper_1310_0041_b200 as gdp
ctx = gdp.Ctx(0)
def t(fn):
    best = None
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = fn(); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = (ms, r) if best is None or ms < best[0] else best
    return best
for cfg in [1]:
    I0 = torch.from_numpy(synth.make_config(cfg)).cuda()
    out = {}
    for fmg in [0, 1, 2, 3]:
        I1 = torch.empty(I0.shape, dtype=torch.float32, device="cuda")
        I2 = torch.empty_like(I1)
        o = gdp.default_opts(fmg=fmg, fmg_slices=fmg)
        ms1, (_, r1) = t(lambda: gdp.gdp_diffuse_z(ctx, I0, I1=I1, opts=o, check=False))
        ms2, (_, r2) = t(lambda: gdp.gdp_screened_poisson_slices(ctx, I0, I1, I2=I2, alpha=0.01, opts=o, check=False))
        print(f"config {cfg} fmg={fmg}: phase1 {ms1:.2f} ms cycles {r1['vcycles']} {['%.2e' % v for v in r1['rel_res']]} {r1['status']}", flush=True)
        print(f"config {cfg} fmg={fmg}: phase2 {ms2:.2f} ms cycles {r2['vcycles']} {['%.2e' % v for v in r2['rel_res']]} {r2['status']}", flush=True)
        out[fmg] = (I1.clone(), I2.clone())
    for k in out:
        d1 = (out[0][0] - out[k][0]).abs().max().item()
        d2 = (out[0][1] - out[k][1]).abs().max().item()
        print(f"config {cfg} fmg={k}: max |I1 diff| {d1:.3e}  max |I2 diff| {d2:.3e}", flush=True)
# per-kernel-class device time of one phase-1 / phase-2 solve on config 1, FMG off / on
I0 = torch.from_numpy(synth.make_config(1)).cuda()
I1 = torch.empty(I0.shape, dtype=torch.float32, device="cuda")
I2 = torch.empty_like(I1)
for fmg in [0, 1, 3]:
    o = gdp.default_opts(fmg=fmg, fmg_slices=fmg)
    for ph in [1, 2]:
        fn = (lambda: gdp.gdp_diffuse_z(ctx, I0, I1=I1, opts=o, check=False)) if ph == 1 else \
             (lambda: gdp.gdp_screened_poisson_slices(ctx, I0, I1, I2=I2, alpha=0.01, opts=o, check=False))
        fn(); torch.cuda.synchronize()
        gdp.profile_begin(); fn(); torch.cuda.synchronize()
        st = gdp.profile_end()
        tot = sum(x["ms"] for x in st)
        print(f"fmg={fmg} phase{ph}: total kernel ms {tot:.2f}, launches {sum(x['launches'] for x in st)}")
        for x in sorted(st, key=lambda x: -x["ms"]):
            print(f"   {x['name']:14s} {x['ms']:7.3f} ms  {x['launches']:5d} launches")
