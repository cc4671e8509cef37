"""Bit-identity of the temporally blocked 3D pass (fused 7) against the per-sweep kernels (3) and
the reference schedule (0) on a few shapes; prints max |diff|."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gdp_synth as synth  # noqa: E402
import paper_1310_0041_b200 as gdp  # noqa: E402

ctx = gdp.Ctx(0)
shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]] or [(16, 64, 64), (33, 130, 252), (12, 1024, 1024)]
for shape in shapes:
    nz, ny, nx = shape
    I0 = torch.from_numpy(synth.make_stack(nx, ny, nz, 41, "u8")).cuda()
    outs = {}
    for fused in (0, 3, 7):
        o = gdp.default_opts(fused=fused, max_vcycles=2, rel_tol=1e-30, stagnation=0, fmg=0)
        I1, rep = gdp.gdp_diffuse_z(ctx, I0, opts=o, check=False)
        torch.cuda.synchronize()
        outs[fused] = I1.cpu().numpy()
    d3 = np.abs(outs[3] - outs[0]).max()
    d7 = np.abs(outs[7] - outs[0]).max()
    bad = np.argwhere(outs[7] != outs[0])
    print(shape, "fused3", d3, "fused7", d7, "nbad", len(bad), bad[:5].tolist(), flush=True)
