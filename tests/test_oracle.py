"""Pins of the CPU oracle (-m "not gpu"): the oracle is checked against things other
than itself — the paper's energies evaluated link by link (brute.py), closed-form cosine
eigenmodes (§3.2), SPEC worked values, invariants and special cases — so that a dropped
term, a wrong sign or index, or a transposed operand fails at least one test."""
import json
import os

import numpy as np
import pytest

import gdp_synth as synth
import oracle as O
from oracle import brute

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RNG = np.random.default_rng(12345)


def _matrix(shape, W, alpha):
    """Dense matrix of oracle.apply_A, column by column."""
    N = int(np.prod(shape))
    A = np.empty((N, N))
    for i in range(N):
        e = np.zeros(N)
        e[i] = 1.0
        A[:, i] = O.apply_A(e.reshape(shape), W, alpha).ravel()
    return A


# ---------------------------------------------------------------- P11 stencil values
def test_stencil_worked_values_spec128():
    g = json.load(open(os.path.join(GOLD, "stencil_spec128.json")))
    shape = (3, 3, 3)
    c = (1 * 3 + 1) * 3 + 1  # centre voxel
    A = _matrix(shape, (1.0, 1.0, 1.0), 0.0)
    assert A[c, c] == pytest.approx(g["W_1_1_1"]["center"])
    for off in (1, 3, 9):
        assert A[c, c + off] == pytest.approx(g["W_1_1_1"]["face"])
        assert A[c, c - off] == pytest.approx(g["W_1_1_1"]["face"])
    A = _matrix(shape, (1.0, 1.0, 0.0), 0.0)
    assert A[c, c] == pytest.approx(g["W_1_1_0"]["center"])
    assert A[c, c + 1] == pytest.approx(g["W_1_1_0"]["inslice_face"])
    assert A[c, c + 9] == pytest.approx(g["W_1_1_0"]["z_face"])
    A = _matrix(shape, (1.0, 1.0, 0.1), 0.0)
    gg = g["W_1_1_0.1"]
    assert A[c, c] == pytest.approx(gg["center"])
    assert A[c, c + 1] == pytest.approx(gg["xy_face"]) and A[c, c - 3] == pytest.approx(gg["xy_face"])
    assert A[c, c + 9] == pytest.approx(gg["z_face"]) and A[c, c - 9] == pytest.approx(gg["z_face"])
    assert A[0, 0] == pytest.approx(gg["corner_diag"])  # Neumann: 2 in-plane links + 1 z link
    assert np.allclose(A.sum(axis=1), 0.0)  # alpha = 0: rows sum to zero
    assert np.allclose(A, A.T)


# ---------------------------------------------------------------- operator == energy Hessian
@pytest.mark.parametrize("shape,W,alpha", [((2, 3, 4), (1.0, 1.0, 0.1), 0.0),
                                           ((3, 3, 2), (0.7, 1.3, 0.25), 0.05),
                                           ((1, 4, 5), (1.0, 1.0, 0.0), 0.01)])
def test_operator_is_energy_hessian(shape, W, alpha):
    V = RNG.random(shape)
    Gx = {}
    # random gradient target on every link (not derived from an image)
    links = brute._links(shape)
    for cc, n, ax in links:
        Gx[(cc, n)] = RNG.standard_normal()
    A_b, b_b = brute.quadratic_form(shape, W, alpha, V=V, G=lambda cc, n, ax: Gx[(cc, n)])
    A_o = _matrix(shape, W, alpha)
    assert np.allclose(A_b, A_o, atol=1e-12)
    # rhs of the oracle for the same targets: G as link arrays
    G = {"x": np.zeros((shape[0], shape[1], shape[2] - 1)), "y": np.zeros((shape[0], shape[1] - 1, shape[2])),
         "z": np.zeros((shape[0] - 1, shape[1], shape[2]))}
    for (cc, n), v in Gx.items():
        ax = [i for i in range(3) if cc[i] != n[i]][0]
        G[{2: "x", 1: "y", 0: "z"}[ax]][cc] = v
    b_o = O.rhs_general(V, G, W, alpha)
    assert np.allclose(b_b, b_o.ravel(), atol=1e-12)


def test_diffusion_rhs_is_energy_linear_term():
    shape = (3, 3, 4)
    I0 = RNG.random(shape)
    W = (1.0, 1.0, 0.1)
    _, b_b = brute.quadratic_form(shape, W, 0.0, G=brute.diffusion_G(I0))
    assert np.allclose(b_b, O.rhs_diffusion(I0, W).ravel(), atol=1e-12)


def test_blend_rhs_is_energy_linear_term():
    shape = (2, 3, 4)
    I0, I1 = RNG.random(shape), RNG.random(shape)
    alpha = 0.01
    for z in range(shape[0]):
        s = (1,) + shape[1:]
        A_b, b_b = brute.quadratic_form(s, (1.0, 1.0, 0.0), alpha, V=I1[z:z + 1],
                                        G=brute.diffusion_G(I0[z:z + 1]))
        b_o = O.rhs_blend(I0[z:z + 1], I1[z:z + 1], alpha)
        assert np.allclose(b_b, b_o.ravel(), atol=1e-12)


# ---------------------------------------------------------------- P1 dense brute force
def test_diffuse_matches_brute_minimiser_tiny():
    shape = (3, 4, 5)
    I0 = RNG.random(shape)
    A, b = brute.quadratic_form(shape, (1.0, 1.0, 0.1), 0.0, G=brute.diffusion_G(I0))
    x = brute.minimiser(A, b, singular_mean=I0.mean())
    assert np.abs(O.diffuse_z(I0).ravel() - x).max() < 1e-8


def test_blend_matches_brute_minimiser_tiny():
    shape = (2, 4, 5)
    I0, I1 = RNG.random(shape), RNG.random(shape)
    alpha = 0.01
    I2 = O.screened_poisson_slices(I0, I1, alpha)
    for z in range(2):
        s = (1, 4, 5)
        A, b = brute.quadratic_form(s, (1.0, 1.0, 0.0), alpha, V=I1[z:z + 1], G=brute.diffusion_G(I0[z:z + 1]))
        assert np.abs(I2[z].ravel() - brute.minimiser(A, b)).max() < 1e-8


def test_dense_solve_16cube():
    """P1 on the largest brute size (<=16^3): CG of the oracle == bordered dense solve."""
    shape = (16, 16, 16)
    I0 = synth.make_stack(16, 16, 16, 99, "f32").astype(np.float64)
    W = (1.0, 1.0, 0.1)
    A = _matrix(shape, W, 0.0)
    b = O.rhs_diffusion(I0, W).ravel()
    N = A.shape[0]
    Bd = np.zeros((N + 1, N + 1))
    Bd[:N, :N] = A
    Bd[:N, N] = 1.0
    Bd[N, :N] = 1.0
    rhs = np.concatenate([b, [I0.sum()]])
    x = np.linalg.solve(Bd, rhs)[:N]
    assert np.abs(O.diffuse_z(I0).ravel() - x).max() < 1e-7


# ---------------------------------------------------------------- P2 closed form
def test_path_eigenvalues_are_spectrum():
    for n in (1, 2, 5, 16):
        mu = O.path_eigenvalues(n)
        for k in range(n):
            v = np.cos(np.pi * k * (np.arange(n) + 0.5) / n)
            Lv = O.apply_A(v.reshape(1, 1, n), (1.0, 0.0, 0.0), 0.0).ravel()
            assert np.allclose(Lv, mu[k] * v, atol=1e-12)


def test_cg_matches_dct_closed_form_config0():
    I0 = synth.make_config(0)
    I1 = O.diffuse_z(I0)
    I1d = O.diffuse_z_dct(I0)
    assert np.abs(I1 - I1d).max() < 1e-8
    I2 = O.screened_poisson_slices(I0, I1, 0.01)
    I2d = O.screened_poisson_slices_dct(I0, I1d, 0.01)
    assert np.abs(I2 - I2d).max() < 1e-8


def test_dct_solve_general():
    shape = (5, 6, 7)
    b = RNG.standard_normal(shape)
    for W, alpha in (((1.0, 2.0, 0.3), 0.1), ((1.0, 1.0, 0.0), 0.5)):
        x = O.dct_solve(b, W, alpha)
        assert np.abs(O.apply_A(x, W, alpha) - b).max() < 1e-10


# ---------------------------------------------------------------- P3 mode gains
def _mode(shape, k, l, m):
    nz, ny, nx = shape
    cx = np.cos(np.pi * k * (np.arange(nx) + 0.5) / nx)
    cy = np.cos(np.pi * l * (np.arange(ny) + 0.5) / ny)
    cz = np.cos(np.pi * m * (np.arange(nz) + 0.5) / nz)
    return cz[:, None, None] * cy[None, :, None] * cx[None, None, :]


def test_mode_101_cube_gain_is_1_over_1p1():
    g = json.load(open(os.path.join(GOLD, "spectral_spec.json")))
    for n in (6, 8):
        phi = _mode((n, n, n), 1, 0, 1)
        I0 = 0.5 + 0.2 * phi
        I1 = O.diffuse_z(I0)
        gain = np.sum((I1 - 0.5) * phi) / np.sum(0.2 * phi * phi)
        assert gain == pytest.approx(1.0 / 1.1, abs=1e-9)
        assert gain == pytest.approx(g["ad_gain_101_cube"], abs=1e-6)


def test_mode_gains_match_discrete_symbols():
    """CG output projected on single cosine modes == §3.2 gains with mu_k = 4 sin^2(pi k/2n)."""
    shape = (16, 64, 64)
    alpha = 0.01
    for (k, l, m) in ((1, 0, 1), (3, 2, 5), (0, 0, 3), (4, 1, 0)):
        phi = _mode(shape, k, l, m)
        I0 = 0.5 + 0.1 * phi
        I1 = O.diffuse_z(I0)
        I2 = O.screened_poisson_slices(I0, I1, alpha)
        nrm = np.sum(0.1 * phi * phi)
        g1 = np.sum((I1 - 0.5) * phi) / nrm
        F = np.sum((I2 - 0.5) * phi) / nrm
        mx = 4 * np.sin(np.pi * k / 128) ** 2
        my = 4 * np.sin(np.pi * l / 128) ** 2
        mz = 4 * np.sin(np.pi * m / 32) ** 2
        g_exp = 1.0 if mx + my + mz == 0 else (mx + my) / (mx + my + 0.1 * mz)
        F_exp = (alpha * g_exp + mx + my) / (alpha + mx + my)
        assert g1 == pytest.approx(g_exp, abs=1e-8)
        assert F == pytest.approx(F_exp, abs=1e-8)
        if m == 0:
            assert g1 == pytest.approx(1.0, abs=1e-8) and F == pytest.approx(1.0, abs=1e-8)
        if k == 0 and l == 0:
            assert g1 == pytest.approx(0.0, abs=1e-8) and F == pytest.approx(0.0, abs=1e-8)


# ---------------------------------------------------------------- P4-P9 invariants
def test_constant_image_unchanged():
    I0 = np.full((4, 8, 8), 0.37)
    I1, I2 = O.destripe(I0)
    assert np.abs(I1 - 0.37).max() < 1e-14 and np.abs(I2 - 0.37).max() < 1e-14


def test_z_invariant_unchanged():
    T = synth.make_stack(24, 20, 1, 5, "f32").astype(np.float64)[0]
    I0 = np.repeat(T[None], 6, axis=0)
    I1, I2 = O.destripe(I0)
    assert np.abs(I1 - I0).max() < 1e-9 and np.abs(I2 - I0).max() < 1e-9


def test_offset_striping_closed_form():
    I0u, T, c = synth.offset_striped_u8(20, 18, 9, 3)
    I1, I2 = O.destripe(I0u)
    exp = O.decode(I0u) - (c[:, None, None] - c.mean()) / 255.0
    exp_exact = (T[None].astype(np.float64) + c.mean()) / 255.0
    # fp32 decode rounding of each input voxel is <= 3e-8
    assert np.abs(exp - exp_exact).max() < 1e-7
    assert np.abs(I1 - exp_exact).max() < 1e-7
    assert np.abs(I2 - exp_exact).max() < 1e-7


def test_dc_invariants():
    I0 = synth.make_stack(32, 24, 8, 11, "u8")
    I1, I2 = O.destripe(I0, alpha=0.05)
    assert I1.mean() == pytest.approx(O.decode(I0).mean(), abs=1e-13)
    assert np.abs(I2.mean(axis=(1, 2)) - I1.mean(axis=(1, 2))).max() < 1e-11


def test_identity_blend():
    I0 = synth.make_stack(20, 16, 3, 4, "f32")
    I2 = O.screened_poisson_slices(I0, O.decode(I0), 0.01)
    assert np.abs(I2 - O.decode(I0)).max() < 1e-9


def test_linearity():
    a = synth.make_stack(16, 12, 5, 1, "f32").astype(np.float64)
    b = synth.make_stack(16, 12, 5, 2, "f32").astype(np.float64)
    fa = O.destripe(a)[1]
    fb = O.destripe(b)[1]
    fab = O.destripe(2.0 * a - 0.5 * b)[1]
    assert np.abs(fab - (2.0 * fa - 0.5 * fb)).max() < 1e-8


def test_limits_paper_bullets():
    """PAPER.md:214-218.  The bullets hold for k^2 + l^2 > 0; the (0,0,m) modes (slice means)
    have gain 0 for every beta_z > 0 and alpha, so in the limits the output is the input with
    its slice means replaced: beta_z -> 0 gives I1 -> I0 - mean_xy(I0) + mean(I0); alpha -> 0
    gives I2 -> I0 - mean_xy(I0) + mean_xy(I1); alpha large gives I2 -> I1."""
    I0 = synth.make_stack(16, 16, 6, 8, "f32").astype(np.float64)
    sm0 = I0.mean(axis=(1, 2), keepdims=True)
    bz = 1e-7
    I1 = O.diffuse_z(I0, W=(1.0, 1.0, bz))
    # deviation of the k^2+l^2>0 modes is <= bz * max(mu_z) / min(mu_xy > 0) * |I0| ~ 1e-5
    assert np.abs(I1 - (I0 - sm0 + I0.mean())).max() < 5e-5
    I1 = O.diffuse_z(I0)
    # alpha = 1e-7: the DC term alpha*mean is ~1e-7 of ||b||, so CG's 1e-10 relative stop
    # resolves it to ~1e-6; smaller alpha would only measure the stopping rule
    I2 = O.screened_poisson_slices(I0, I1, 1e-7)
    assert np.abs(I2 - (I0 - sm0 + I1.mean(axis=(1, 2), keepdims=True))).max() < 2e-6
    I2 = O.screened_poisson_slices(I0, I1, 1e6)
    assert np.abs(I2 - I1).max() < 1e-4
    # discrete filter bounded in [0, 1]
    mu = RNG.random((3, 1000)) * 4
    F = O.combined_gain(mu[0], mu[1], mu[2], 0.01)
    assert F.min() >= 0.0 and F.max() <= 1.0 + 1e-15


def test_residual_x0_is_b_and_exact_is_zero():
    shape = (4, 5, 6)
    b = RNG.standard_normal(shape)
    W = (1.0, 1.0, 0.1)
    assert np.array_equal(O.residual(np.zeros(shape), b, W, 0.3), b)
    x = O.dct_solve(b, W, 0.3)
    assert O.rel_residual(x, b, W, 0.3) < 1e-12


def test_decode_is_fp32_division():
    u = np.arange(256, dtype=np.uint8)
    d = O.decode(u)
    assert np.array_equal(d, (u.astype(np.float32) / np.float32(255)).astype(np.float64))
    assert d[0] == 0.0 and d[255] == 1.0


# ---------------------------------------------------------------- P3 worked values (golden)
def _p3_cases():
    g = json.load(open(os.path.join(GOLD, "spectral_p3.json")))
    return g["tol"], g["cases"]


def _symbols(shape, mode):
    (nz, ny, nx), (k, l, m) = shape, mode
    return O.path_eigenvalues(nx)[k], O.path_eigenvalues(ny)[l], O.path_eigenvalues(nz)[m]


@pytest.mark.parametrize("i", range(5))
def test_p3_golden_gain_functions(i):
    """closed_form.ad_gain / combined_gain / sp_gain reproduce SURVEY §8(c) P3's printed values
    (a swapped numerator, a dropped alpha or a z symbol in the SP term fails one of them)."""
    tol, cases = _p3_cases()
    c = cases[i]
    mx, my, mz = _symbols(c["shape"], c["mode"])
    assert float(O.ad_gain(mx, my, mz)) == pytest.approx(c["g_ad"], abs=tol)
    assert float(O.combined_gain(mx, my, mz, c["alpha"])) == pytest.approx(c["F"], abs=tol)
    if "sp_I1_only" in c:
        assert float(O.sp_gain(mx, my, c["alpha"])) == pytest.approx(c["sp_I1_only"], abs=tol)


@pytest.mark.parametrize("i", range(5))
def test_p3_golden_gains_measured_by_cg(i):
    """The CG oracle's outputs projected onto the mode give the same P3 values."""
    tol, cases = _p3_cases()
    c = cases[i]
    shape, (k, l, m), alpha = tuple(c["shape"]), c["mode"], c["alpha"]
    phi = _mode(shape, k, l, m)
    I0 = 0.5 + 0.1 * phi
    nrm = np.sum(0.1 * phi * phi)
    I1 = O.diffuse_z(I0)
    assert np.sum((I1 - 0.5) * phi) / nrm == pytest.approx(c["g_ad"], abs=tol)
    I2 = O.screened_poisson_slices(I0, I1, alpha)
    assert np.sum((I2 - 0.5) * phi) / nrm == pytest.approx(c["F"], abs=tol)
    if "sp_I1_only" in c:  # a mode present in I1 only: I0 constant
        J2 = O.screened_poisson_slices(np.full(shape, 0.5), I0, alpha)
        assert np.sum((J2 - 0.5) * phi) / nrm == pytest.approx(c["sp_I1_only"], abs=tol)
        # the DCT phase-2 solver agrees on the same input
        J2d = O.screened_poisson_slices_dct(np.full(shape, 0.5), I0, alpha)
        assert np.abs(J2d - J2).max() < 1e-9


def test_sp_gain_is_dct_phase2_transfer():
    """sp_gain(mu_k, mu_l, alpha) is the transfer of screened_poisson_slices_dct for a mode of I1
    (the full-size GPU tests use it as their expected value)."""
    shape = (3, 24, 40)
    alpha = 0.03
    for (k, l) in ((1, 0), (5, 7), (0, 11), (39, 23)):
        phi = _mode(shape, k, l, 0)
        J2 = O.screened_poisson_slices_dct(np.zeros(shape), phi, alpha)
        mx, my, _ = _symbols(shape, (k, l, 0))
        g = np.sum(J2 * phi) / np.sum(phi * phi)
        assert g == pytest.approx(float(O.sp_gain(mx, my, alpha)), abs=1e-12)
        # and the dense matrix of the 2D operator has that mode as an eigenvector
    A = _matrix((1, 6, 5), (1.0, 1.0, 0.0), alpha)
    ev = np.sort(np.linalg.eigvalsh(A))
    mus = np.sort((O.path_eigenvalues(5)[None, :] + O.path_eigenvalues(6)[:, None]).ravel())
    assert np.allclose(ev, alpha + mus, atol=1e-12)
    assert np.allclose(np.sort(alpha / ev), np.sort(O.sp_gain(mus, 0.0, alpha)), atol=1e-12)


def test_slice_rel_residuals_hand_built():
    """Per-slice ||b_i - A x_i|| / ||b_i|| on slices whose residual follows from the 2D
    stencil values alone (centre 4 + alpha, faces -1, corner 2 + alpha)."""
    alpha = 0.25
    nz, ny, nx = 4, 5, 6
    x = np.zeros((nz, ny, nx))
    b = np.zeros((nz, ny, nx))
    x[0] = 0.7                     # constant: L x = 0, A x = alpha x = b exactly
    b[0] = alpha * 0.7
    b[1] = RNG.standard_normal((ny, nx))  # x = 0: residual = b, rel = 1
    x[2, 2, 3] = 1.0               # interior delta, b = 0: r = -A e, ||r||^2 = (4+alpha)^2 + 4
    x[3, 0, 0] = 1.0               # corner delta (2 links), b = (2+alpha) e: r = e_right + e_up
    b[3, 0, 0] = 2.0 + alpha
    rel = O.slice_rel_residuals(x, b, alpha)
    assert rel[0] == pytest.approx(0.0, abs=1e-15)
    assert rel[1] == pytest.approx(1.0, abs=1e-15)
    assert rel[2] == pytest.approx(np.sqrt((4 + alpha) ** 2 + 4), abs=1e-14)  # ||b|| = 0: absolute
    assert rel[3] == pytest.approx(np.sqrt(2.0) / (2.0 + alpha), abs=1e-15)


def test_decode_correctly_rounded_rationals():
    """decode(u) is the fp32 value nearest to the rational u/255 (ties to even), checked with
    exact rational arithmetic on every code — not by re-dividing in fp32."""
    from fractions import Fraction
    d = O.decode(np.arange(256, dtype=np.uint8))
    for u in range(256):
        f = np.float32(d[u])
        assert float(f) == d[u]  # an fp32 value
        q = Fraction(u, 255)
        err = abs(Fraction(float(f)) - q)
        for nb in (np.nextafter(f, np.float32(-1)), np.nextafter(f, np.float32(2))):
            e2 = abs(Fraction(float(nb)) - q)
            assert err < e2 or (err == e2 and (f.view(np.uint32) & 1) == 0)
    assert d[51] == float(np.float32(0.2)) and d[0] == 0.0 and d[255] == 1.0
