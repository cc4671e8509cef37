"""Ad-hoc GPU diagnostics (not a test): convergence histories and timings."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gdp_synth as synth
import paper_1310_0041_b200 as gdp

ctx = gdp.Ctx(0)
def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()
for shape, dt in [((16, 64, 64), "f32"), ((9, 63, 65), "u8"), ((128, 1024, 1024), "u8")]:
    nz, ny, nx = shape
    t = time.time(); I0 = synth.make_stack(nx, ny, nz, 1, dt); tg = time.time() - t
    I0d = dev(I0)
    for fused in (0,):
        o = gdp.default_opts(fused=fused)
        for rep_i in range(2):
            torch.cuda.synchronize(); t = time.time()
            I1, I2, r1, r2 = gdp.gdp_destripe(gdp.Ctx.__new__(gdp.Ctx) if False else ctx, I0d, opts=o)
            torch.cuda.synchronize(); el = time.time() - t
        print(shape, dt, "gen %.1fs" % tg, "wall %.2f ms" % (el * 1e3))
        for r in (r1, r2):
            print("   ", r["status"], "levels", r["levels"], "cyc", r["vcycles"], "dev %.2f ms" % (r["seconds"] * 1e3),
                  "launch", r["kernel_launches"], " ".join("%.1e" % v for v in r["rel_res"]))
        N = nx * ny * nz
        print("   voxels/s %.3e" % (N / (r1["seconds"] + r2["seconds"])))
