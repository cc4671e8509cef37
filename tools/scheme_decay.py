"""NEXT-3 convergence study in the style of the paper's Fig. 3: per-V-cycle
residual decay and device time of the Constant (this library's main path), Hybrid and Linear
discretisations on the synthetic config stack, both phases.  Prints one JSON line per scheme.

    python tools/scheme_decay.py [config] [nz] [nu_pre nu_post]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gdp_synth as synth
import paper_1310_0041_b200 as gdp

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
nz = (int(sys.argv[2]) or None) if len(sys.argv) > 2 else None
nu = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else None
ctx = gdp.Ctx(0)
I0 = torch.from_numpy(synth.make_config(cfg, nz=nz)).cuda()
for scheme in ("constant", "hybrid", "linear"):
    kw = dict(scheme=scheme, rel_tol=1e-7, max_vcycles=12, stagnation=0, dx_tol=0.0)
    if scheme == "constant":
        kw.update(fmg=0, fmg_slices=0)  # plain V-cycles from x0 for the decay comparison
    if nu:
        kw.update(nu_pre=nu[0], nu_post=nu[1], nu_pre_slices=nu[0], nu_post_slices=nu[1])
    o = gdp.default_opts(**kw)
    for _ in range(2):  # the first solve builds the hierarchy
        I1, I2, r1, r2 = gdp.gdp_destripe(ctx, I0, alpha=0.01, opts=o)
    torch.cuda.synchronize()
    out = {"scheme": scheme, "dims": list(I0.shape), "nu": [o.nu_pre, o.nu_post, o.nu_pre_slices, o.nu_post_slices]}
    for ph, r in (("phase1", r1), ("phase2", r2)):
        rr = r["rel_res"]
        dec = [rr[k + 1] / rr[k] for k in range(len(rr) - 1) if rr[k] > 0]
        out[ph] = {"vcycles": r["vcycles"], "levels": r["levels"], "rel_res": rr, "ms": r["seconds"] * 1e3,
                   "decay_per_cycle": dec,
                   "mean_decay": float(np.exp(np.mean(np.log(dec)))) if dec else None,
                   "ms_per_cycle": r["seconds"] * 1e3 / max(r["vcycles"], 1)}
    print(json.dumps(out), flush=True)
ctx.close()
