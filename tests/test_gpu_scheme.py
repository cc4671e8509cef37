"""GPU parity (-m gpu) of NEXT-3, the paper's Hybrid and Linear discretisations,
through the C ABI against the oracle (oracle/fem_linear.py for Linear and for the Galerkin
hierarchy; oracle/gdp_oracle.py for Hybrid, whose finest system is the Constant one).

Bars as tests/test_gpu_parity.py: solutions within 5e-5 per phase (1e-4 end to end), relative
residual <= 1e-6 evaluated by the oracle in fp64; operators (every Galerkin level) within fp32
rounding of the oracle's fp64 sparse products: |y_gpu - y| <= 64 eps32 (|A| |x|)."""
import os

import numpy as np
import pytest
import torch

import gdp_synth as synth
import oracle as O
from oracle import fem_linear as FL
import paper_1310_0041_b200 as gdp

pytestmark = pytest.mark.gpu

TOL_X = 5e-5
TOL_R = 1e-6
W_AD = (1.0, 1.0, 0.1)
EPS32 = 2.0 ** -24


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def host(t):
    return t.detach().cpu().numpy().astype(np.float64)


def _fine(scheme, shape, W, alpha, per_slice):
    if scheme == "linear":
        return FL.tensor_operator(shape, W, alpha, per_slice=per_slice)
    return FL.tensor_operator(shape, W, alpha, FL.identity_1d, FL.fd_1d, per_slice=per_slice)


@pytest.mark.parametrize("scheme", ["hybrid", "linear"])
@pytest.mark.parametrize("shape,W,alpha,per_slice", [((9, 40, 37), W_AD, 0.0, False),
                                                     ((16, 70, 66), (1.0, 0.5, 1.0), 0.2, False),
                                                     ((3, 130, 99), (1.0, 1.0, 0.0), 0.01, True),
                                                     ((2, 1, 150), (1.0, 1.0, 0.0), 0.1, True)])
def test_galerkin_levels_match_oracle(gpu_ctx, scheme, shape, W, alpha, per_slice):
    """Every level operator = P^T ... A ... P assembled by the oracle (reading L-4)."""
    opts = gdp.default_opts(coarse_max=64)
    lv = gdp.gdp_scheme_levels(gpu_ctx, scheme, shape, W, alpha, per_slice, opts=opts)
    assert len(lv) >= 3 and tuple(lv[0]["dims"]) == shape
    hier = FL.hierarchy(shape, _fine(scheme, shape, W, alpha, per_slice), [l["coarsened"] for l in lv[1:]])
    rng = np.random.default_rng(7)
    for l, (s, A) in enumerate(hier):
        assert tuple(lv[l]["dims"]) == s
        x = rng.random(s).astype(np.float32)
        y = host(gdp.gdp_scheme_apply(gpu_ctx, scheme, l, dev(x), fine_dims=shape, W=W, alpha=alpha,
                                      per_slice=per_slice, opts=opts))
        ref = (A @ x.astype(np.float64).ravel()).reshape(s)
        bound = 64 * EPS32 * (abs(A) @ np.abs(x.astype(np.float64)).ravel()).reshape(s) + 1e-30
        assert np.all(np.abs(y - ref) <= bound), (l, np.abs(y - ref).max(), bound.max())


@pytest.mark.parametrize("shape", [(9, 40, 37), (1, 1, 1), (4, 1, 70), (33, 20, 2)])
def test_hybrid_phase1_matches_constant_oracle(gpu_ctx, shape):
    I0 = synth.make_stack(shape[2], shape[1], shape[0], 3, "u8")
    I1, rep = gdp.gdp_diffuse_z(gpu_ctx, torch.from_numpy(I0).cuda(), opts=gdp.default_opts(scheme="hybrid"))
    assert rep["status"] == "GDP_OK", rep
    ref = O.diffuse_z(I0)
    x = host(I1)
    assert np.abs(x - ref).max() <= TOL_X
    assert abs(x.mean() - O.decode(I0).mean()) <= 1e-6
    b = O.rhs_diffusion(O.decode(I0), W_AD)
    if np.linalg.norm(b) > 0:
        assert O.rel_residual(x, b, W_AD, 0.0) <= TOL_R


@pytest.mark.parametrize("shape,alpha", [((5, 70, 61), 0.01), ((2, 129, 128), 0.001), ((3, 17, 1), 0.1)])
def test_hybrid_phase2_matches_constant_oracle(gpu_ctx, shape, alpha):
    I0 = synth.make_stack(shape[2], shape[1], shape[0], 4, "u8")
    I1 = O.diffuse_z(I0).astype(np.float32)
    I2, rep = gdp.gdp_screened_poisson_slices(gpu_ctx, torch.from_numpy(I0).cuda(), dev(I1), alpha=alpha,
                                              opts=gdp.default_opts(scheme="hybrid"))
    assert rep["status"] == "GDP_OK", rep
    ref = O.screened_poisson_slices(I0, I1.astype(np.float64), alpha)
    x = host(I2)
    assert np.abs(x - ref).max() <= TOL_X
    b = O.rhs_blend(O.decode(I0), I1.astype(np.float64), alpha)
    # reading c-12: the gate is 1e-6 or the fp32 representation floor of the slice, whichever is
    # larger (a 17 x 1 slice with a small ||b|| has |A||x| / ||b|| ~ 50: floor ~ 1e-6)
    floor = 4 * 2.0 ** -24 * np.sqrt((((alpha + 8.0) * np.abs(x)) ** 2).sum(axis=(1, 2))) / \
        np.sqrt((b ** 2).sum(axis=(1, 2)))
    assert np.all(O.slice_rel_residuals(x, b, alpha) <= np.maximum(TOL_R, floor))


@pytest.mark.parametrize("shape", [(9, 40, 37), (1, 1, 1), (4, 1, 70), (12, 33, 34)])
def test_linear_phase1_matches_fem_oracle(gpu_ctx, shape):
    I0 = synth.make_stack(shape[2], shape[1], shape[0], 5, "u8")
    I1, rep = gdp.gdp_diffuse_z(gpu_ctx, torch.from_numpy(I0).cuda(), opts=gdp.default_opts(scheme="linear"))
    assert rep["status"] == "GDP_OK", rep
    ref = FL.diffuse_z_linear(I0)
    x = host(I1)
    assert np.abs(x - ref).max() <= TOL_X
    b = FL.rhs_diffusion_linear(I0)
    if np.abs(b).max() > 1e-12:
        assert FL.rel_residual_linear(x, b - b.mean(), W_AD, 0.0) <= TOL_R


@pytest.mark.parametrize("shape,alpha", [((5, 70, 61), 0.01), ((2, 129, 128), 0.001), ((3, 17, 1), 0.1)])
def test_linear_phase2_matches_fem_oracle(gpu_ctx, shape, alpha):
    I0 = synth.make_stack(shape[2], shape[1], shape[0], 6, "u8")
    I1 = FL.diffuse_z_linear(I0).astype(np.float32)
    I2, rep = gdp.gdp_screened_poisson_slices(gpu_ctx, torch.from_numpy(I0).cuda(), dev(I1), alpha=alpha,
                                              opts=gdp.default_opts(scheme="linear"))
    assert rep["status"] == "GDP_OK", rep
    ref = FL.screened_poisson_slices_linear(I0, I1.astype(np.float64), alpha)
    x = host(I2)
    assert np.abs(x - ref).max() <= TOL_X
    b = FL.rhs_blend_linear(I0, I1.astype(np.float64), alpha)
    assert FL.slice_rel_residuals_linear(x, b, alpha).max() <= TOL_R


@pytest.mark.parametrize("scheme", ["hybrid", "linear"])
def test_scheme_destripe_end_to_end(gpu_ctx, scheme):
    I0 = synth.make_config(0)  # config 0: 64 x 64 x 16 fp32
    I1, I2, r1, r2 = gdp.gdp_destripe(gpu_ctx, torch.from_numpy(I0).cuda(), alpha=0.01,
                                      opts=gdp.default_opts(scheme=scheme))
    if scheme == "linear":
        ref1, ref2 = FL.destripe_linear(I0, 0.01)
    else:
        ref1, ref2 = O.destripe(I0, 0.01)
    assert np.abs(host(I1) - ref1).max() <= TOL_X
    assert np.abs(host(I2) - ref2).max() <= 2 * TOL_X


@pytest.mark.parametrize("scheme", ["hybrid", "linear"])
def test_scheme_vcycle_and_residual_api(gpu_ctx, scheme):
    """gdp_vcycle with opts.scheme contracts the scheme's own residual; gdp_scheme_residual is
    the oracle's b - A x."""
    shape = (10, 48, 50)
    rng = np.random.default_rng(8)
    A = _fine(scheme, shape, W_AD, 0.05, False)
    xs = rng.random(shape)
    b = (A @ xs.ravel()).reshape(shape)
    x = torch.zeros(shape, dtype=torch.float32, device="cuda")
    bd = dev(b)
    o = gdp.default_opts(scheme=scheme)
    rels = [gdp.gdp_vcycle(gpu_ctx, x, bd, W=W_AD, alpha=0.05, opts=o) for _ in range(4)]
    assert rels[0] < 0.2 and all(r1 < r0 for r0, r1 in zip(rels, rels[1:]))
    r, rr, bb = gdp.gdp_scheme_residual(gpu_ctx, scheme, x, bd, torch.empty_like(x), W=W_AD, alpha=0.05)
    ref = b.astype(np.float32).astype(np.float64) - (A @ host(x).ravel()).reshape(shape)
    assert np.abs(host(r) - ref).max() <= 64 * EPS32 * (np.abs(b).max() + 10 * np.abs(host(x)).max())
    assert rr == pytest.approx((host(r) ** 2).sum(), rel=1e-6)  # fp64 sum of the fp32 residual


def test_scheme_rejects_distributed_and_npr(gpu_ctx):
    ctx = gdp.Ctx(0, loopback=2)
    I0 = torch.from_numpy(synth.make_stack(16, 16, 4, 0, "u8")).cuda()
    with pytest.raises(gdp.GdpError):
        gdp.gdp_npr_filter(gpu_ctx, I0, opts=gdp.default_opts(scheme="linear"))
    with pytest.raises(gdp.GdpError):
        gdp.gdp_diffuse_z(ctx, I0, opts=gdp.default_opts(scheme="hybrid"))
    ctx.close()


_REF_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import gdp_synth as synth, paper_1310_0041_b200 as gdp
ctx = gdp.Ctx(0)
out = {{}}
for scheme in ("hybrid", "linear"):
    for shape in {shapes!r}:
        I0 = torch.from_numpy(synth.make_stack(shape[2], shape[1], shape[0], 9, "u8")).cuda()
        I1, I2, r1, r2 = gdp.gdp_destripe(ctx, I0, alpha=0.01, opts=gdp.default_opts(scheme=scheme))
        out[f"{{scheme}}_{{shape}}_1"] = I1.cpu().numpy()
        out[f"{{scheme}}_{{shape}}_2"] = I2.cpu().numpy()
np.savez({path!r}, **out)
"""


def test_tiled_half_sweeps_bit_identical_to_colour_launches(gpu_ctx, tmp_path):
    """The shared-memory tiled half-sweeps of the 27-point levels (k_ts_gs_tile, opt-in with
    GDP_TS_TILE=1) reproduce the default one-launch-per-colour sweeps bit for bit (same colour
    order, same per-cell arithmetic); each variant runs in a subprocess of its own."""
    import subprocess
    import sys
    shapes = [(12, 100, 90), (7, 257, 131), (33, 64, 72)]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for tile in ("0", "1"):
        path = str(tmp_path / f"out{tile}.npz")
        env = dict(os.environ, GDP_TS_TILE=tile)
        subprocess.run([sys.executable, "-c", _REF_SCRIPT.format(root=root, shapes=shapes, path=path)], env=env,
                       check=True, timeout=600)
        outs.append(np.load(path))
    for key in outs[0].files:
        assert np.array_equal(outs[0][key], outs[1][key]), key
