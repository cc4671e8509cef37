"""Per-cycle change ||x_k - x_{k-1}||_inf of both phases on the config-1 stack (the a9 / H3
correction-norm test): the solve is rerun with max_vcycles = k (stagnation off, tiny rel_tol),
which returns the iterate after exactly k cycles."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import gdp_synth as synth
import paper_1310_0041_b200 as gdp

ctx = gdp.Ctx(0)
I0 = torch.from_numpy(synth.make_config(1)).cuda()
prev = None
for k in range(1, 6):
    o = gdp.default_opts(max_vcycles=k, rel_tol=1e-12, stagnation=0)
    I1, r = gdp.gdp_diffuse_z(ctx, I0, opts=o)
    torch.cuda.synchronize()
    d = float((I1 - prev).abs().max()) if prev is not None else float("nan")
    print(f"phase1 k={k} rel={r['rel_res'][k]:.3e} max|dx|={d:.3e}", flush=True)
    prev = I1.clone()
I1 = prev
for alpha in (0.001, 0.01, 0.1):
    prev = None
    for k in range(1, 6):
        o = gdp.default_opts(max_vcycles=k, rel_tol=1e-12, stagnation=0)
        I2, r = gdp.gdp_screened_poisson_slices(ctx, I0, I1, alpha=alpha, opts=o)
        torch.cuda.synchronize()
        d = float((I2 - prev).abs().max()) if prev is not None else float("nan")
        print(f"phase2 a={alpha} k={k} rel={r['rel_res'][k]:.3e} max|dx|={d:.3e}", flush=True)
        prev = I2.clone()
