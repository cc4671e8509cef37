"""GPU parity (-m gpu): the CUDA path, called through the C ABI, against the CPU oracle on
the same seeded inputs.

Bars (BASELINE.json north_star):
  * solutions: max |x_gpu - x_oracle| <= 1e-4 on [0,1] intensities; each phase is held to
    5e-5 so the two-phase pipeline stays within 1e-4 (reading c-13);
  * residual: ||b - A x_gpu|| / ||b|| <= 1e-6, evaluated by the oracle in fp64 against the
    oracle's fp64 b (phase 2: every slice);
  * the residual kernel itself: |r_gpu - r_fp64| <= 8 eps32 * (|b| + sum_links |coef| (|x_c|+|x_n|)
    + alpha |x|) per voxel (fp32 rounding of <= 16 operations).
"""
import numpy as np
import pytest
import torch

import gdp_synth as synth
import oracle as O
import paper_1310_0041_b200 as gdp

pytestmark = pytest.mark.gpu

TOL_X = 5e-5
TOL_R = 1e-6
W_AD = (1.0, 1.0, 0.1)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.detach().cpu().numpy().astype(np.float64)


def _rel_ad(I0, I1_gpu, W=W_AD):
    b = O.rhs_diffusion(O.decode(I0) if I0.dtype != np.float64 else I0, W)
    return O.rel_residual(I1_gpu, b, W, 0.0)


def _rel_sp(I0, I1, I2_gpu, alpha):
    b = O.rhs_blend(O.decode(I0), I1, alpha)
    return O.slice_rel_residuals(I2_gpu, b, alpha).max()


# ------------------------------------------------------------------ a1 decode
def test_u8_decode_is_ieee_division(gpu_ctx):
    """rel_tol = 1e30 returns x0 = decode(I0) untouched (the mean pin shift is exactly 0)."""
    u = np.arange(256, dtype=np.uint8).reshape(1, 1, 256)
    I1, rep = gdp.gdp_diffuse_z(gpu_ctx, dev(u), opts=gdp.default_opts(rel_tol=1e30))
    assert rep["vcycles"] == 0
    exp = np.arange(256, dtype=np.float32) / np.float32(255.0)
    assert np.array_equal(I1.cpu().numpy().ravel(), exp)


# ------------------------------------------------------------------ residual kernel
@pytest.mark.parametrize("shape,W,alpha", [((7, 33, 45), (1.0, 1.0, 0.1), 0.0),
                                           ((3, 64, 64), (0.5, 2.0, 0.3), 0.25),
                                           ((1, 17, 130), (1.0, 1.0, 0.0), 0.01),
                                           ((5, 1, 9), (1.0, 1.0, 1.0), 0.0)])
def test_residual_elementwise(gpu_ctx, shape, W, alpha):
    rng = np.random.default_rng(3)
    x = rng.random(shape).astype(np.float32)
    b = (rng.random(shape) * 2 - 1).astype(np.float32)
    r = torch.empty(shape, dtype=torch.float32, device="cuda")
    _, nr, nb = gdp.gdp_residual(gpu_ctx, dev(x), dev(b), r, W=W, alpha=alpha)
    r64 = O.residual(x.astype(np.float64), b.astype(np.float64), W, alpha)
    coef = 2 * (W[0] + W[1] + W[2]) + alpha
    bound = 8 * 2.0 ** -24 * (np.abs(b) + coef * 2 * np.abs(x).max() + 1.0)
    assert np.all(np.abs(host(r) - r64) <= bound)
    assert nr == pytest.approx(np.sum(r64 * r64), rel=1e-5)
    assert nb == pytest.approx(np.sum(b.astype(np.float64) ** 2), rel=1e-12)


# ------------------------------------------------------------------ phase 1
@pytest.mark.parametrize("shape,dtype,seed", [((16, 64, 64), "f32", 0),      # config 0
                                              ((9, 63, 65), "u8", 5),
                                              ((5, 37, 29), "f32", 6),
                                              ((33, 40, 48), "u8", 7),
                                              ((2, 200, 150), "u8", 8)])
def test_diffuse_z_parity(gpu_ctx, shape, dtype, seed):
    nz, ny, nx = shape
    I0 = synth.make_stack(nx, ny, nz, seed, dtype)
    I1, rep = gdp.gdp_diffuse_z(gpu_ctx, dev(I0))
    assert rep["status"] == "GDP_OK", rep
    ref = O.diffuse_z(I0)
    x = host(I1)
    assert np.abs(x - ref).max() <= TOL_X
    assert _rel_ad(I0, x) <= TOL_R
    assert x.mean() == pytest.approx(O.decode(I0).mean(), abs=1e-6)


# ------------------------------------------------------------------ phase 2
@pytest.mark.parametrize("alpha", [0.001, 0.01, 0.1])
@pytest.mark.parametrize("shape,dtype", [((4, 96, 128), "u8"), ((3, 65, 47), "f32"), ((2, 300, 260), "u8")])
def test_screened_poisson_parity(gpu_ctx, shape, dtype, alpha):
    nz, ny, nx = shape
    I0 = synth.make_stack(nx, ny, nz, 21, dtype)
    I1 = O.diffuse_z(I0).astype(np.float32)  # phase 2 checked in isolation (reading c-13)
    I2, rep = gdp.gdp_screened_poisson_slices(gpu_ctx, dev(I0), dev(I1), alpha=alpha)
    assert rep["status"] == "GDP_OK", rep
    ref = O.screened_poisson_slices(I0, I1, alpha)
    x = host(I2)
    assert np.abs(x - ref).max() <= TOL_X
    assert _rel_sp(I0, I1, x, alpha) <= TOL_R


def test_destripe_config0(gpu_ctx):
    I0 = synth.make_config(0)
    I1, I2, r1, r2 = gdp.gdp_destripe(gpu_ctx, dev(I0), alpha=0.01)
    ref1, ref2 = O.destripe(I0, alpha=0.01)
    assert np.abs(host(I1) - ref1).max() <= TOL_X
    assert np.abs(host(I2) - ref2).max() <= 1e-4
    assert r1["status"] == "GDP_OK" and r2["status"] == "GDP_OK"


# ------------------------------------------------------------------ closed forms / edge cases
def test_constant_stack_is_fixed_point(gpu_ctx):
    I0 = np.full((6, 40, 52), 77, np.uint8)
    I1, I2, r1, r2 = gdp.gdp_destripe(gpu_ctx, dev(I0))
    v = np.float32(77) / np.float32(255)
    assert np.all(host(I1) == v) and np.all(host(I2) == v)


def test_offset_striping_closed_form(gpu_ctx):
    I0, T, c = synth.offset_striped_u8(256, 256, 32, 2)
    exp = (T[None].astype(np.float64) + c.mean()) / 255.0
    I1, I2, r1, r2 = gdp.gdp_destripe(gpu_ctx, dev(I0))
    assert np.abs(host(I1) - exp).max() <= TOL_X
    assert np.abs(host(I2) - exp).max() <= 1e-4


def test_single_slice_and_thin(gpu_ctx):
    for shape in ((1, 70, 90), (2, 3, 200), (4, 1, 1), (1, 1, 1)):
        nz, ny, nx = shape
        I0 = synth.random_field(shape, 4)
        I1, rep = gdp.gdp_diffuse_z(gpu_ctx, dev(I0))
        ref = O.diffuse_z(I0)
        assert np.abs(host(I1) - ref).max() <= TOL_X, shape
        I1f = ref.astype(np.float32)
        I2, rep = gdp.gdp_screened_poisson_slices(gpu_ctx, dev(I0), dev(I1f), alpha=0.01)
        assert np.abs(host(I2) - O.screened_poisson_slices(I0, I1f, 0.01)).max() <= TOL_X, shape


def test_vcycle_and_residual_api(gpu_ctx):
    shape = (8, 48, 40)
    rng = np.random.default_rng(9)
    for W, alpha in ((W_AD, 0.0), ((1.0, 1.0, 1.0), 0.05)):
        b = rng.standard_normal(shape)
        if alpha == 0.0:
            b -= b.mean()
        b32 = b.astype(np.float32)
        x = torch.zeros(shape, dtype=torch.float32, device="cuda")
        rels = [gdp.gdp_vcycle(gpu_ctx, x, dev(b32), W=W, alpha=alpha) for _ in range(8)]
        assert all(r1 < r0 for r0, r1 in zip(rels[:3], rels[1:4]))
        assert rels[-1] < 1e-5
        ref = O.dct_solve(b32.astype(np.float64), W, alpha)
        xs = host(x)
        if alpha == 0.0:
            xs -= xs.mean()
        assert np.abs(xs - ref).max() < 1e-4 * max(1.0, np.abs(ref).max())


def test_invalid_arguments(gpu_ctx):
    I0 = dev(np.zeros((2, 8, 8), np.uint8))
    with pytest.raises(gdp.GdpError) as e:
        gdp.gdp_diffuse_z(gpu_ctx, I0, W=(-1.0, 1.0, 0.1))
    assert e.value.code == 1
    with pytest.raises(gdp.GdpError) as e:
        gdp.gdp_diffuse_z(gpu_ctx, I0, W=(0.0, 0.0, 0.0), alpha=0.0)
    assert e.value.code == 1
    I1 = torch.zeros((2, 8, 8), dtype=torch.float32, device="cuda")
    with pytest.raises(gdp.GdpError) as e:
        gdp.gdp_screened_poisson_slices(gpu_ctx, I0, I1, alpha=0.0)
    assert e.value.code == 1


def test_report_and_launches(gpu_ctx):
    I0 = synth.make_config(0)
    before = gdp.kernel_launch_count()
    I1, rep = gdp.gdp_diffuse_z(gpu_ctx, dev(I0))
    assert rep["levels"] >= 2 and 1 <= rep["vcycles"] <= 12
    assert rep["rel_res"][-1] <= 1e-6 and rep["rel_res"][0] > 1e-3
    assert rep["kernel_launches"] > 0 and gdp.kernel_launch_count() - before == rep["kernel_launches"]
    assert rep["seconds"] > 0


# ------------------------------------------------------------------ schedules agree bit for bit
@pytest.mark.parametrize("shape,dtype,alpha", [((3, 130, 260), "u8", 0.01), ((2, 75, 61), "f32", 0.1),
                                               ((1, 517, 389), "u8", 0.001), ((4, 64, 64), "u8", 0.01),
                                               ((16, 1024, 1024), "u8", 0.01), ((3, 1031, 777), "f32", 0.01)])
def test_fused_2d_bit_identical_to_reference(gpu_ctx, shape, dtype, alpha):
    nz, ny, nx = shape
    I0 = synth.make_stack(nx, ny, nz, 31, dtype)
    I1 = dev(O.diffuse_z_dct(I0).astype(np.float32))
    outs = []
    for fused in (0, 1, 9):  # reference, fused 2D passes, + the cooperative coarse tail
        o = gdp.default_opts(fused=fused, max_vcycles=3, rel_tol=1e-30, stagnation=0)
        I2, rep = gdp.gdp_screened_poisson_slices(gpu_ctx, dev(I0), I1, alpha=alpha, opts=o, check=False)
        outs.append(I2.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(outs[0], outs[2])


def test_fused_2d_vcycle_bit_identical(gpu_ctx):
    shape = (2, 190, 157)
    rng = np.random.default_rng(5)
    b = dev(rng.standard_normal(shape).astype(np.float32))
    xs = []
    for fused in (0, 1):
        x = torch.zeros(shape, dtype=torch.float32, device="cuda")
        for _ in range(2):
            gdp.gdp_vcycle(gpu_ctx, x, b, W=(1.0, 0.5, 0.0), alpha=0.05, opts=gdp.default_opts(fused=fused, nu_pre=1, nu_post=2))
        xs.append(x.cpu().numpy())
    assert np.array_equal(xs[0], xs[1])


@pytest.mark.parametrize("shape,dtype", [((16, 64, 64), "f32"), ((9, 63, 65), "u8"), ((33, 130, 250), "u8"),
                                         ((24, 517, 389), "u8"), ((12, 1024, 1024), "u8"), ((67, 150, 300), "u8"),
                                         ((128, 256, 200), "u8"), ((40, 200, 180), "f32"), ((3, 300, 260), "f32")])
def test_fused_3d_bit_identical_to_reference(gpu_ctx, shape, dtype):
    nz, ny, nx = shape
    I0 = synth.make_stack(nx, ny, nz, 41, dtype)
    outs = []
    # reference, one kernel per sweep, one kernel per pass (temporal blocking), + cooperative coarse
    # tail, the vertical-pack z-march
    reps = []
    for fused in (0, 3, 7, 11, 35, 34):
        o = gdp.default_opts(fused=fused, max_vcycles=2, rel_tol=1e-30, stagnation=0)
        I1, rep = gdp.gdp_diffuse_z(gpu_ctx, dev(I0), opts=o, check=False)
        outs.append(I1.cpu().numpy())
        reps.append(rep)
    for k in range(1, len(outs)):
        assert np.array_equal(outs[0], outs[k]), k
        # the reported residual history too (norm sums in another order, the fused tails adding
        # up to 32 squares per thread in fp32 before fp64: relative 1e-6)
        n = reps[0]["vcycles"] + 1
        assert reps[k]["vcycles"] == reps[0]["vcycles"], k
        np.testing.assert_allclose(reps[k]["rel_res"][:n], reps[0]["rel_res"][:n], rtol=1e-6, atol=0)


@pytest.mark.parametrize("nu", [(1, 1), (2, 1), (1, 2), (2, 2), (3, 1)])
@pytest.mark.parametrize("shape", [(10, 70, 90), (21, 132, 260)])
def test_fused_3d_vcycle_nu_variants(gpu_ctx, nu, shape):
    rng = np.random.default_rng(11)
    b = rng.standard_normal(shape)
    b -= b.mean()
    bd = dev(b.astype(np.float32))
    xs = []
    for fused in (0, 3, 7, 11, 35):
        x = torch.zeros(shape, dtype=torch.float32, device="cuda")
        for _ in range(2):
            gdp.gdp_vcycle(gpu_ctx, x, bd, W=(1.0, 1.0, 0.1), alpha=0.0,
                           opts=gdp.default_opts(fused=fused, nu_pre=nu[0], nu_post=nu[1]))
        xs.append(x.cpu().numpy())
    for k in range(1, len(xs)):
        assert np.array_equal(xs[0], xs[k]), k


# ------------------------------------------------------------------ z-slab partition (loopback)
@pytest.mark.parametrize("shape,world", [((16, 64, 64), 2), ((33, 40, 48), 3), ((128, 96, 96), 4),
                                         ((12, 70, 90), 5), ((64, 130, 75), 8)])
@pytest.mark.parametrize("fmg", [0, 1])
def test_loopback_partition_bit_identical(gpu_ctx, shape, world, fmg):
    """Phase 1 on `world` z-slabs (halo exchange per half-sweep, gathered coarse levels, the FMG
    start level by level) gives the single-rank iterate bit for bit, and the oracle's answer."""
    nz, ny, nx = shape
    I0 = synth.make_stack(nx, ny, nz, 51, "u8")
    o = gdp.default_opts(fused=0, fmg=fmg)
    ref, r1 = gdp.gdp_diffuse_z(gpu_ctx, dev(I0), opts=o)
    lb = gdp.Ctx(0, loopback=world)
    try:
        out, r2 = gdp.gdp_diffuse_z(lb, dev(I0), opts=o)
    finally:
        lb.close()
    # norms are fp64 sums in different orders (fused initial residual vs per-slab partials)
    assert r1["vcycles"] == r2["vcycles"]
    assert np.allclose(r1["rel_res"], r2["rel_res"], rtol=1e-6, atol=0)
    assert np.array_equal(ref.cpu().numpy(), out.cpu().numpy())
    assert np.abs(host(out) - O.diffuse_z(I0)).max() <= TOL_X


@pytest.mark.parametrize("shape,world", [((48, 128, 256), 2), ((40, 130, 250), 4), ((128, 256, 256), 8),
                                         ((27, 96, 200), 3)])
@pytest.mark.parametrize("fmg", [0, 1])
def test_loopback_fused_partition_bit_identical(gpu_ctx, shape, world, fmg):
    """Default opts: the finest level of every slab runs the fused z-march sweeps with 3 ghost
    planes per face (and the FMG start on the team); the iterate equals the single-rank fused
    solve bit for bit, in the same number of cycles."""
    nz, ny, nx = shape
    I0 = synth.make_stack(nx, ny, nz, 53, "u8")
    o = gdp.default_opts(fmg=fmg)
    ref, r1 = gdp.gdp_diffuse_z(gpu_ctx, dev(I0), opts=o)
    lb = gdp.Ctx(0, loopback=world)
    try:
        out, r2 = gdp.gdp_diffuse_z(lb, dev(I0), opts=o)
    finally:
        lb.close()
    assert r1["vcycles"] == r2["vcycles"]
    assert np.allclose(r1["rel_res"], r2["rel_res"], rtol=1e-6, atol=0)
    assert np.array_equal(ref.cpu().numpy(), out.cpu().numpy())


def test_loopback_destripe_and_slices(gpu_ctx):
    I0 = synth.make_stack(80, 72, 20, 52, "u8")
    o = gdp.default_opts(fused=0, fmg=0, fmg_slices=0)
    a = gdp.gdp_destripe(gpu_ctx, dev(I0), opts=o)
    lb = gdp.Ctx(0, loopback=4)
    try:
        b = gdp.gdp_destripe(lb, dev(I0), opts=o)
    finally:
        lb.close()
    assert np.array_equal(a[1].cpu().numpy(), b[1].cpu().numpy())


# ------------------------------------------------------------------ a13 out-of-core streamer
@pytest.mark.parametrize("shape,dtype,pin", [((40, 180, 200), "u8", True), ((33, 130, 250), "f32", False),
                                             ((18, 256, 256), "u8", True)])
def test_out_of_core_matches_in_core(gpu_ctx, shape, dtype, pin):
    """A 1-byte HBM budget forces the streamer (finest level on the host, two-plane z-windows,
    slice batches of one): phase 1 is bit-identical to the in-core solve (same kernels per
    voxel, same per-plane mean-pin sums), phase 2 (per-batch stopping) meets the same bars."""
    nz, ny, nx = shape
    I0 = synth.make_stack(nx, ny, nz, 61, dtype)
    t0 = torch.from_numpy(I0)
    if pin:
        t0 = t0.pin_memory()
    outs = []
    for budget in (0, 1):
        I1 = torch.empty(shape, dtype=torch.float32)
        I2 = torch.empty(shape, dtype=torch.float32)
        if pin:
            I1, I2 = I1.pin_memory(), I2.pin_memory()
        # the streamer has no FMG start (gdp.h); compare like with like
        r1, r2 = gdp.gdp_destripe_host(gpu_ctx, t0, I2, I1=I1, alpha=0.01, hbm_budget_bytes=budget,
                                       opts=gdp.default_opts(fmg=0, fmg_slices=0))
        assert r1["status"] == "GDP_OK" and r2["status"] == "GDP_OK", (budget, r1, r2)
        outs.append((I1.numpy().copy(), I2.numpy().copy(), r1, r2))
    (a1, a2, ra, _), (b1, b2, rb, rb2) = outs
    assert ra["vcycles"] == rb["vcycles"]
    assert np.array_equal(a1, b1)
    ref1, ref2 = O.destripe(I0, alpha=0.01)
    assert np.abs(b1 - ref1).max() <= TOL_X
    assert np.abs(b2 - ref2).max() <= 1e-4
    assert np.abs(a2 - b2).max() <= 2e-5
    assert _rel_sp(I0, ref1, b2.astype(np.float64), 0.01) <= 2 * TOL_R
    assert rb["hbm_bytes_est"] > 0  # host-link bytes of the streamed finest level


@pytest.mark.parametrize("shape,budget,fuse", [((5, 96, 100), 1, 1), ((7, 64, 80), 1, 0),
                                               ((64, 512, 512), 300 << 20, 1), ((64, 512, 512), 300 << 20, 0)])
def test_out_of_core_stream_fusion_bit_identical(gpu_ctx, shape, budget, fuse):
    """NEXT-2: multi-sweep streaming passes (z-lagged stages, cross-cycle fusion) and one pass per
    sweep give the in-core phase-1 iterate bit for bit, for stacks shorter than the stage lag and
    for windows wider than it (a 300 MB budget: 4-plane chunks of 512^2)."""
    nz, ny, nx = shape
    I0 = synth.make_stack(nx, ny, nz, 62, "u8")
    t0 = torch.from_numpy(I0).pin_memory()
    outs = []
    for b in (0, budget):
        I1 = torch.empty(shape, dtype=torch.float32).pin_memory()
        I2 = torch.empty(shape, dtype=torch.float32).pin_memory()
        r1, r2 = gdp.gdp_destripe_host(gpu_ctx, t0, I2, I1=I1, alpha=0.01, hbm_budget_bytes=b,
                                       opts=gdp.default_opts(fmg=0, fmg_slices=0, stream_fuse=fuse))
        assert r1["status"] == "GDP_OK" and r2["status"] == "GDP_OK", (b, r1, r2)
        outs.append((I1.numpy().copy(), r1))
    (a1, ra), (b1, rb) = outs
    assert rb["hbm_bytes_est"] > 0 and ra["vcycles"] == rb["vcycles"]
    assert np.array_equal(a1, b1)


@pytest.mark.parametrize("budget_mb", [1600, 2000])
def test_out_of_core_partial_residency(gpu_ctx, budget_mb):
    """a13 partial residency: a budget below the in-core need (~2.1 GB for 96 x 1024^2 u8) keeps as
    many planes of the iterate in HBM as it can (1.6 GB: about half of them; 2.0 GB: all, and I0):
    the iterate stays bit-identical to the in-core solve and fewer bytes cross the host link than
    when everything streams."""
    shape = (96, 1024, 1024)
    I0 = synth.make_stack(shape[2], shape[1], shape[0], 63, "u8")
    t0 = torch.from_numpy(I0).pin_memory()
    outs = []
    for b in (0, budget_mb << 20, 1):
        I1 = torch.empty(shape, dtype=torch.float32).pin_memory()
        I2 = torch.empty(shape, dtype=torch.float32).pin_memory()
        r1, r2 = gdp.gdp_destripe_host(gpu_ctx, t0, I2, I1=I1, alpha=0.01, hbm_budget_bytes=b,
                                       opts=gdp.default_opts(fmg=0, fmg_slices=0))
        assert r1["status"] == "GDP_OK" and r2["status"] == "GDP_OK", (b, r1, r2)
        outs.append((I1.numpy().copy(), r1))
    (a1, ra), (p1, rp), (s1, rs) = outs
    assert ra["vcycles"] == rp["vcycles"] == rs["vcycles"]
    assert np.array_equal(a1, p1) and np.array_equal(a1, s1)
    assert 0 < rp["hbm_bytes_est"] < rs["hbm_bytes_est"]
    # without a caller I1 the streamer pins a scratch for the non-resident planes only: same I2
    I2a = torch.empty(shape, dtype=torch.float32).pin_memory()
    I2b = torch.empty(shape, dtype=torch.float32).pin_memory()
    o = gdp.default_opts(fmg=0, fmg_slices=0)
    gdp.gdp_destripe_host(gpu_ctx, t0, I2a, I1=torch.empty(shape, dtype=torch.float32).pin_memory(), alpha=0.01,
                          hbm_budget_bytes=budget_mb << 20, opts=o)
    gdp.gdp_destripe_host(gpu_ctx, t0, I2b, alpha=0.01, hbm_budget_bytes=budget_mb << 20, opts=o)
    assert torch.equal(I2a, I2b)


# ------------------------------------------------------------------ NEXT-1: the §6 NPR filter
@pytest.mark.parametrize("shape,dtype,params", [((16, 135, 240), "u8", (0.001, 1.25, 5 / 255)),
                                                ((9, 63, 65), "f32", (0.01, 1.0, 0.05)),
                                                ((24, 100, 300), "u8", (0.001, 1.25, 5 / 255))])
def test_npr_filter_parity(gpu_ctx, shape, dtype, params):
    """General 3D screened solve with a modulated gradient field against the
    oracle's CG; residual against the oracle's fp64 rhs."""
    alpha, lam, sigma = params
    nz, ny, nx = shape
    I0 = synth.make_stack(nx, ny, nz, 71, dtype)
    out, rep = gdp.gdp_npr_filter(gpu_ctx, dev(I0), alpha=alpha, lam=lam, sigma=sigma)
    assert rep["status"] == "GDP_OK", rep
    ref = O.npr_filter(I0, W=W_AD, alpha=alpha, lam=lam, sigma=sigma)
    x = host(out)
    assert np.abs(x - ref).max() <= TOL_X
    b = O.rhs_npr(O.decode(I0), W_AD, alpha, lam, sigma)
    assert O.rel_residual(x, b, W_AD, alpha) <= TOL_R


def test_npr_filter_limits_and_errors(gpu_ctx):
    I0 = synth.make_stack(40, 30, 5, 72, "f32")
    x, _ = gdp.gdp_npr_filter(gpu_ctx, dev(I0), alpha=0.001, lam=1.0, sigma=1e-9)  # identity filter
    assert np.abs(host(x) - I0.astype(np.float64)).max() <= 1e-5
    c = np.full((4, 20, 24), 0.4, np.float32)
    x, _ = gdp.gdp_npr_filter(gpu_ctx, dev(c))  # constant volume unchanged
    assert np.abs(host(x) - 0.4).max() <= 1e-7
    for kw in (dict(alpha=0.0), dict(sigma=0.0), dict(lam=-1.0)):
        with pytest.raises(gdp.GdpError):
            gdp.gdp_npr_filter(gpu_ctx, dev(I0), **kw)


# ------------------------------------------------------------------ FMG start (gdp_opts.fmg)
@pytest.mark.parametrize("shape,W,fmg,dtype,nu", [((24, 517, 389), (1.0, 1.0, 0.1), 1, "u8", (2, 2)),
                                                   ((33, 130, 250), (1.0, 1.0, 0.1), 2, "u8", (2, 2)),
                                                   ((40, 200, 180), (1.0, 1.0, 0.1), 3, "u8", (2, 2)),
                                                   ((32, 96, 96), (1.0, 1.0, 1.0), 1, "u8", (2, 2)),
                                                   ((12, 1024, 1024), (1.0, 1.0, 0.1), 1, "u8", (2, 2)),
                                                   ((19, 131, 203), (1.0, 1.0, 0.1), 1, "f32", (2, 2)),
                                                   ((21, 140, 180), (1.0, 1.0, 0.1), 1, "u8", (1, 2))])
def test_fmg_phase1_schedules_bit_identical(gpu_ctx, shape, W, fmg, dtype, nu):
    """The FMG start gives the same iterate in the reference and fused schedules, and with r0
    restricted inside the init pass or by the restriction kernel (fmg + 4); nu_pre = 1 takes
    the prolongation kernel at the finest level instead of the first fused sweep."""
    nz, ny, nx = shape
    I0 = synth.make_stack(nx, ny, nz, 43, dtype)
    outs = []
    for fused, f in ((0, fmg), (3, fmg), (3, fmg + 4), (7, fmg), (7, fmg + 4), (11, fmg), (35, fmg), (35, fmg + 4)):
        o = gdp.default_opts(fused=fused, fmg=f, max_vcycles=2, rel_tol=1e-30, stagnation=0,
                             nu_pre=nu[0], nu_post=nu[1])
        I1, rep = gdp.gdp_diffuse_z(gpu_ctx, dev(I0), W=W, opts=o, check=False)
        outs.append(I1.cpu().numpy())
    for k in range(1, len(outs)):
        assert np.array_equal(outs[0], outs[k]), k


@pytest.mark.parametrize("shape,fmg,dtype", [((3, 1031, 777), 1, "u8"), ((16, 1024, 1024), 3, "u8"),
                                              ((2, 300, 260), 2, "u8"), ((4, 517, 389), 3, "f32")])
def test_fmg_phase2_schedules_bit_identical(gpu_ctx, shape, fmg, dtype):
    nz, ny, nx = shape
    I0 = synth.make_stack(nx, ny, nz, 47, dtype)
    I1 = dev(O.diffuse_z_dct(I0).astype(np.float32))
    outs = []
    for fused, f in ((0, fmg), (1, fmg), (1, fmg + 4), (9, fmg)):
        o = gdp.default_opts(fused=fused, fmg_slices=f, max_vcycles=2, rel_tol=1e-30, stagnation=0)
        I2, rep = gdp.gdp_screened_poisson_slices(gpu_ctx, dev(I0), I1, alpha=0.01, opts=o, check=False)
        outs.append(I2.cpu().numpy())
    for k in range(1, len(outs)):
        assert np.array_equal(outs[0], outs[k]), k


@pytest.mark.parametrize("fmg", [1, 2, 3])
def test_fmg_converges_to_oracle(gpu_ctx, fmg):
    """Same stopping rule, same converged answer as the oracle (and fewer or equal cycles)."""
    I0 = synth.make_stack(96, 80, 24, 7, "u8")
    ref1, ref2 = O.destripe(I0, alpha=0.01)
    o = gdp.default_opts(fmg=fmg, fmg_slices=fmg)
    I1, I2, r1, r2 = gdp.gdp_destripe(gpu_ctx, dev(I0), alpha=0.01, opts=o)
    _, _, p1, p2 = gdp.gdp_destripe(gpu_ctx, dev(I0), alpha=0.01, opts=gdp.default_opts(fmg=0, fmg_slices=0))
    assert r1["rel_res"][-1] <= 1e-6 and r2["rel_res"][-1] <= 1e-6
    assert r1["vcycles"] <= p1["vcycles"] and r2["vcycles"] <= p2["vcycles"]
    assert np.abs(host(I1) - ref1).max() <= TOL_X
    assert np.abs(host(I2) - ref2).max() <= 1e-4


# ------------------------------------------------------------------ building blocks on a z-slab partition
@pytest.mark.parametrize("shape,world,W,alpha", [((16, 64, 64), 2, W_AD, 0.0), ((33, 40, 48), 3, W_AD, 0.0),
                                                 ((64, 130, 75), 8, W_AD, 0.0), ((24, 70, 90), 4, (1.0, 0.5, 0.3), 0.05)])
def test_loopback_vcycle_and_residual_match_single_rank(gpu_ctx, shape, world, W, alpha):
    """gdp_vcycle / gdp_residual on a loopback partition (halo exchange per half-sweep, gathered coarse
    levels, per-plane fp64 sums in global order) equal the single-rank calls (reference schedule)."""
    rng = np.random.default_rng(13)
    b = rng.standard_normal(shape)
    if alpha == 0.0:
        b -= b.mean()
    bd = dev(b.astype(np.float32))
    o = gdp.default_opts(fused=0)
    lb = gdp.Ctx(0, loopback=world)
    try:
        xs, rels = [], []
        for ctx in (gpu_ctx, lb):
            x = torch.zeros(shape, dtype=torch.float32, device="cuda")
            rel = [gdp.gdp_vcycle(ctx, x, bd, W=W, alpha=alpha, opts=o) for _ in range(2)]
            xs.append(x.cpu().numpy())
            rels.append(rel)
        assert np.array_equal(xs[0], xs[1])
        assert np.allclose(rels[0], rels[1], rtol=1e-12, atol=0)
        # the residual of that iterate, elementwise and its norms
        x = dev(xs[0])
        outs = []
        for ctx in (gpu_ctx, lb):
            r = torch.empty(shape, dtype=torch.float32, device="cuda")
            _, nr, nb = gdp.gdp_residual(ctx, x, bd, r=r, W=W, alpha=alpha)
            outs.append((r.cpu().numpy(), nr, nb))
        assert np.array_equal(outs[0][0], outs[1][0])
        assert outs[0][1] == pytest.approx(outs[1][1], rel=1e-12) and outs[0][2] == pytest.approx(outs[1][2], rel=1e-12)
        ref = O.residual(xs[0].astype(np.float64), b.astype(np.float32).astype(np.float64), W, alpha)
        assert np.abs(outs[1][0] - ref).max() <= 1e-5 * (1.0 + np.abs(ref).max())
    finally:
        lb.close()


def test_loopback_unaligned_z_coarsening_rejected(gpu_ctx):
    """W = (1, 1, 1) coarsens z from level 0; 33 planes over 3 slabs leaves slabs on odd planes, which the
    gathered restriction cannot map: a clean GDP_EINVAL (never uninitialised coarse planes)."""
    I0 = synth.make_stack(48, 40, 33, 57, "u8")
    lb = gdp.Ctx(0, loopback=3)
    try:
        with pytest.raises(gdp.GdpError) as ei:
            gdp.gdp_diffuse_z(lb, dev(I0), W=(1.0, 1.0, 1.0), opts=gdp.default_opts(fmg=0))
        assert ei.value.code == 1
        # an even split of the same stack works and matches the single-rank solve
        I0e = I0[:32]
        ref, _ = gdp.gdp_diffuse_z(gpu_ctx, dev(I0e), W=(1.0, 1.0, 1.0), opts=gdp.default_opts(fused=0, fmg=0))
        lb2 = gdp.Ctx(0, loopback=2)
        try:
            out, _ = gdp.gdp_diffuse_z(lb2, dev(I0e), W=(1.0, 1.0, 1.0), opts=gdp.default_opts(fused=0, fmg=0))
        finally:
            lb2.close()
        assert np.array_equal(ref.cpu().numpy(), out.cpu().numpy())
    finally:
        lb.close()


# ------------------------------------------------------------------ a9 correction-norm gate (dx_tol)
def test_dx_tol_gate_measures_last_correction(gpu_ctx):
    """The report's dx_inf is ||x_k - x_{k-1}||_inf of the last cycle (checked against two solves
    stopped one cycle apart), and a tight dx_tol keeps the solve going past the residual gate."""
    I0 = dev(synth.make_stack(256, 192, 24, 61, "u8"))
    I1, rep = gdp.gdp_diffuse_z(gpu_ctx, I0)
    k = rep["vcycles"]
    assert rep["status"] == "GDP_OK" and 0.0 <= rep["dx_inf"] <= 1e-4 and rep["rel_res"][-1] <= 1e-6
    prev, _ = gdp.gdp_diffuse_z(gpu_ctx, I0, opts=gdp.default_opts(max_vcycles=k - 1, rel_tol=1e-30, stagnation=0,
                                                                   dx_tol=0.0), check=False)
    # the mean pin adds one scalar per solve: compare the correction, not the pinned outputs
    d = (I1 - prev).cpu().numpy().astype(np.float64)
    exact = np.abs(d - np.mean(d)).max()
    assert rep["dx_inf"] == pytest.approx(exact, rel=0.05, abs=2e-7)
    tight, rep2 = gdp.gdp_diffuse_z(gpu_ctx, I0, opts=gdp.default_opts(dx_tol=1e-7, stagnation=0))
    assert rep2["vcycles"] > k and rep2["dx_inf"] >= 0.0
    off, rep3 = gdp.gdp_diffuse_z(gpu_ctx, I0, opts=gdp.default_opts(dx_tol=0.0))
    assert rep3["dx_inf"] == -1.0 or rep3["vcycles"] <= k


def test_cuda_graph_replay_bit_identical(gpu_ctx):
    """use_graphs: the V-cycles of later solves replay captured CUDA graphs (same launches counted),
    with the same iterate, report and launch count as plain launches."""
    I0 = dev(synth.make_stack(320, 256, 20, 63, "u8"))
    st = torch.cuda.Stream()
    outs = {}
    for g in (0, 1):
        o = gdp.default_opts(use_graphs=g)
        res = []
        for _ in range(3):  # the first solve warms the hierarchy, the next ones capture / replay
            I1, I2, r1, r2 = gdp.gdp_destripe(gpu_ctx, I0, alpha=0.01, opts=o, stream=st)
            st.synchronize()
            res.append((I1.cpu().numpy(), I2.cpu().numpy(), r1, r2))
        outs[g] = res
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        assert a[2]["rel_res"] == b[2]["rel_res"] and a[3]["rel_res"] == b[3]["rel_res"]
        assert a[2]["kernel_launches"] == b[2]["kernel_launches"] and a[3]["kernel_launches"] == b[3]["kernel_launches"]


def test_host_entry_in_core_batched_phase2(gpu_ctx):
    """gdp_destripe_host in core, phase 2 in slice batches (GDP_E2E_BATCHES, default 1) whose
    device-to-host copies overlap the next batch's solve.  Slices are independent systems, so the
    result meets the same bars as the one-launch device solve."""
    shape = (96, 140, 200)
    nz, ny, nx = shape
    I0 = synth.make_stack(nx, ny, nz, 65, "u8")
    t0 = torch.from_numpy(I0).pin_memory()
    I1 = torch.empty(shape, dtype=torch.float32).pin_memory()
    I2 = torch.empty(shape, dtype=torch.float32).pin_memory()
    r1, r2 = gdp.gdp_destripe_host(gpu_ctx, t0, I2, I1=I1, alpha=0.01)
    assert r1["status"] == "GDP_OK" and r2["status"] == "GDP_OK"
    d1, d2, _, _ = gdp.gdp_destripe(gpu_ctx, dev(I0), alpha=0.01)
    assert np.array_equal(I1.numpy(), d1.cpu().numpy())  # phase 1 is the same solve
    assert np.abs(I2.numpy() - d2.cpu().numpy()).max() <= 2e-5
    ref1, ref2 = O.destripe(I0, alpha=0.01)
    assert np.abs(I2.numpy().astype(np.float64) - ref2).max() <= 1e-4
    assert _rel_sp(I0, I1.numpy().astype(np.float64), I2.numpy().astype(np.float64), 0.01) <= TOL_R
