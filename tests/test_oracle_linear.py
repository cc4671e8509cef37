"""Pins of the NEXT-3 oracle (oracle/fem_linear.py, -m "not gpu"), each against something other
than the oracle's own formula:
  * the Linear matrices and right-hand sides against the paper's energies
    integrated by Gauss quadrature of the B-spline interpolants (basis values and gradients
    evaluated at the quadrature points — not the element matrices);
  * closed-form DCT-I eigenmodes of the Neumann hat basis (symbols 2 - 2cos t and (2 + cos t)/3,
    derived by hand below), including the mean pin;
  * the B-spline nesting: on an odd axis the Galerkin coarse operators are the finite-element
    matrices of the coarse hats (spacing 2: mass x 2, stiffness / 2);
  * transfer invariants (constants, ramps, the Fig. 2 pair of PAPER.md:296-301) and the tensor
    identity P^T (A (x) B) P = (P^T A P) (x) (P^T B P) against brute-force sparse products;
  * CG solutions against dense solves, and the invariants of the method (constant / z-invariant
    stacks are fixed points, identity blend)."""
import itertools

import numpy as np
import pytest

import gdp_synth as synth
import oracle as O
from oracle import fem_linear as L

GAUSS = (0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0))  # 2-point Gauss-Legendre on [0, 1]


def _quadrature_operators(shape, per_slice=False):
    """Basis values / partial derivatives of the trilinear (bilinear per slice) interpolant at
    every Gauss point, and the point weights.  Returns (val, {axis: grad}, w): val and grad are
    (Q x N) matrices, N = nodes; x_h(q) = val @ x, d x_h / d axis (q) = grad[axis] @ x."""
    nz, ny, nx = shape
    N = nx * ny * nz

    def elems(n):
        return [(i, 1.0) for i in range(n - 1)] if n > 1 else [(0, None)]

    rows_v, rows_g, wts = [], {a: [] for a in "xyz"}, []
    zel = [(k, None) for k in range(nz)] if per_slice else elems(nz)
    for (k, kz), (j, ky), (i, kx) in itertools.product(zel, elems(ny), elems(nx)):
        pts = [(GAUSS if kx else (0.0,)), (GAUSS if ky else (0.0,)), (GAUSS if kz else (0.0,))]
        for tx, ty, tz in itertools.product(*pts):
            w = (0.5 if kx else 1.0) * (0.5 if ky else 1.0) * (0.5 if kz else 1.0)
            v = np.zeros(N)
            g = {a: np.zeros(N) for a in "xyz"}
            # the 8 (or fewer) corner nodes of the element and their trilinear hats
            for cx, cy, cz in itertools.product((0, 1) if kx else (0,), (0, 1) if ky else (0,),
                                                (0, 1) if kz else (0,)):
                hx = (tx if cx else 1.0 - tx) if kx else 1.0
                hy = (ty if cy else 1.0 - ty) if ky else 1.0
                hz = (tz if cz else 1.0 - tz) if kz else 1.0
                dx = ((1.0 if cx else -1.0) if kx else 0.0)
                dy = ((1.0 if cy else -1.0) if ky else 0.0)
                dz = ((1.0 if cz else -1.0) if kz else 0.0)
                n = ((k + cz) * ny + (j + cy)) * nx + (i + cx)
                v[n] += hx * hy * hz
                g["x"][n] += dx * hy * hz
                g["y"][n] += hx * dy * hz
                g["z"][n] += hx * hy * dz
            rows_v.append(v)
            for a in "xyz":
                rows_g[a].append(g[a])
            wts.append(w)
    return np.array(rows_v), {a: np.array(r) for a, r in rows_g.items()}, np.array(wts)


def _energy_system(shape, W, alpha, per_slice, target_grad_of=None, target_val=None):
    """(A, b) of E(x) = int sum_d beta_d (d_d x_h - G_d)^2 + alpha (x_h - V_h)^2 dp,
    written as E = x^T A x - 2 b^T x + c, by quadrature.  G = grad of target_grad_of's
    interpolant in x and y (the paper's G of Eq. (1) / (2)), V = target_val's interpolant."""
    val, grad, w = _quadrature_operators(shape, per_slice)
    N = val.shape[1]
    A = np.zeros((N, N))
    b = np.zeros(N)
    beta = {"x": W[0], "y": W[1], "z": 0.0 if per_slice else W[2]}
    for a in "xyz":
        if beta[a] == 0.0:
            continue
        Gw = grad[a] * w[:, None]
        A += beta[a] * grad[a].T @ Gw
        if target_grad_of is not None and a in "xy":
            b += beta[a] * Gw.T @ (grad[a] @ target_grad_of.ravel())
    if alpha:
        Vw = val * w[:, None]
        A += alpha * val.T @ Vw
        if target_val is not None:
            b += alpha * Vw.T @ (val @ target_val.ravel())
    return A, b


@pytest.mark.parametrize("shape", [(3, 4, 5), (2, 3, 2), (1, 3, 4)])
def test_linear_phase1_matrix_and_rhs_are_the_energy(shape):
    W = (1.0, 0.7, 0.1)
    I0 = np.random.default_rng(3).random(shape)
    A_q, b_q = _energy_system(shape, W, 0.0, False, target_grad_of=I0)
    A = L.linear_operator(shape, W, 0.0).toarray()
    np.testing.assert_allclose(A, A_q, atol=1e-13)
    np.testing.assert_allclose(L.rhs_diffusion_linear(I0, W).ravel(), b_q, atol=1e-13)


@pytest.mark.parametrize("shape", [(2, 4, 5), (3, 3, 1)])
def test_linear_phase2_matrix_and_rhs_are_the_energy(shape):
    alpha = 0.37
    rng = np.random.default_rng(4)
    I0, I1 = rng.random(shape), rng.random(shape)
    A_q, b_q = _energy_system(shape, (1.0, 1.0, 0.0), alpha, True, target_grad_of=I0, target_val=I1)
    A = L.linear_operator(shape, (1.0, 1.0, 0.0), alpha, per_slice=True).toarray()
    np.testing.assert_allclose(A, A_q, atol=1e-13)
    np.testing.assert_allclose(L.rhs_blend_linear(I0, I1, alpha).ravel(), b_q, atol=1e-13)


def test_1d_matrices_on_nodal_functions():
    # int over [0, n-1] of 1 is n-1; of x is (n-1)^2/2; int (x')^2 of x is n-1 (hand values)
    for n in (2, 3, 7):
        one = np.ones(n)
        ramp = np.arange(n, dtype=float)
        assert one @ L.mass_1d(n) @ one == pytest.approx(n - 1)
        assert one @ L.mass_1d(n) @ ramp == pytest.approx((n - 1) ** 2 / 2)
        assert ramp @ L.mass_1d(n) @ ramp == pytest.approx((n - 1) ** 3 / 3)
        assert ramp @ L.stiff_1d(n) @ ramp == pytest.approx(n - 1)
        assert np.abs(L.stiff_1d(n) @ one).max() == 0.0


# ---------------------------------------------------------------- DCT-I closed forms
def _mode(shape, k):
    nz, ny, nx = shape
    cx = np.cos(np.pi * k[0] * np.arange(nx) / (nx - 1))
    cy = np.cos(np.pi * k[1] * np.arange(ny) / (ny - 1))
    cz = np.cos(np.pi * k[2] * np.arange(nz) / (nz - 1))
    return cz[:, None, None] * cy[None, :, None] * cx[None, None, :]


def _ratio(k, n):
    """mu / lambda of a DCT-I mode: K v = (2 - 2 cos t) D v and M v = (2 + cos t)/3 D v with
    D = diag(1/2, 1, ..., 1, 1/2), t = pi k / (n - 1) (interior rows: cos(t(i-1)) + cos(t(i+1)) =
    2 cos t cos(ti); end rows by the half weight)."""
    t = np.pi * k / (n - 1)
    return (2.0 - 2.0 * np.cos(t)) / ((2.0 + np.cos(t)) / 3.0)


@pytest.mark.parametrize("k", [(1, 0, 0), (2, 3, 1), (0, 1, 2), (5, 1, 3)])
def test_linear_phase1_cosine_mode_gain(k):
    shape, W = (6, 9, 11), (1.0, 1.0, 0.1)
    v = _mode(shape, k)
    I1 = L.diffuse_z_linear(v, W)
    sx, sy, sz = _ratio(k[0], 11), _ratio(k[1], 9), _ratio(k[2], 6)
    g = (W[0] * sx + W[1] * sy) / (W[0] * sx + W[1] * sy + W[2] * sz)
    expect = g * v + (1.0 - g) * v.mean()  # the mean pin adds the constant that restores mean(I0)
    np.testing.assert_allclose(I1, expect, atol=1e-8)


@pytest.mark.parametrize("k", [(1, 0), (3, 2), (7, 5)])
def test_linear_phase2_cosine_mode_gains(k):
    shape, alpha = (2, 9, 12), 0.05
    v = _mode((2, 9, 12), (k[0], k[1], 0))
    s = _ratio(k[0], 12) + _ratio(k[1], 9)
    low = L.screened_poisson_slices_linear(np.zeros(shape), v, alpha)    # I1 = v, I0 = 0
    high = L.screened_poisson_slices_linear(v, np.zeros(shape), alpha)   # I0 = v, I1 = 0
    np.testing.assert_allclose(low, alpha / (alpha + s) * v, atol=1e-9)
    np.testing.assert_allclose(high, s / (alpha + s) * v, atol=1e-9)


# ---------------------------------------------------------------- transfers / Galerkin
@pytest.mark.parametrize("n", [3, 5, 9, 17])
def test_galerkin_is_the_coarse_spline_basis_on_odd_axes(n):
    P = L.prolongation_1d(n)
    nc = (n + 1) // 2
    np.testing.assert_allclose(L.galerkin(L.mass_1d(n), P).toarray(), 2.0 * L.mass_1d(nc).toarray(), atol=1e-14)
    np.testing.assert_allclose(L.galerkin(L.stiff_1d(n), P).toarray(), 0.5 * L.stiff_1d(nc).toarray(), atol=1e-14)
    # SPEC example: interior rows of P^T (-1, 2, -1) P keep the second-difference shape
    Kc = L.galerkin(L.fd_1d(n), P).toarray()
    if nc >= 3:
        np.testing.assert_allclose(Kc[1, :3], [-0.5, 1.0, -0.5])


@pytest.mark.parametrize("n", [2, 4, 6, 7, 10])
def test_prolongation_reproduces_constants_and_ramps(n):
    P = L.prolongation_1d(n)
    nc = (n + 1) // 2
    np.testing.assert_array_equal(P @ np.ones(nc), np.ones(n))
    ramp = P @ (2.0 * np.arange(nc))
    expect = np.arange(n, dtype=float)
    if n % 2 == 0:
        expect[-1] = n - 2  # reading L-4: the last odd node copies its only parent
    np.testing.assert_array_equal(ramp, expect)
    for A in (L.fd_1d(n), L.stiff_1d(n)):
        assert np.abs(L.galerkin(A, P) @ np.ones(nc)).max() < 1e-14  # null space kept


def test_fig2_pair_survives_linear_restriction():
    # a -1/+1 feature inside one coarse cell cancels under (1,1) but not under
    # the B-spline restriction R = P^T
    r = np.zeros(12)
    r[4], r[5] = 1.0, -1.0
    box = np.zeros((6, 12))
    for I in range(6):
        box[I, 2 * I] = box[I, 2 * I + 1] = 1.0
    assert np.abs(box @ r).max() == 0.0
    Rr = L.prolongation_1d(12).T @ r
    np.testing.assert_allclose(Rr[2:4], [0.5, -0.5])


def test_prolongation_matches_spline_nesting_pointwise():
    # hat(t/2) = 1/2 hat(t+1) + hat(t) + 1/2 hat(t-1): evaluate the coarse hat centred on fine
    # node 2I at fine node i directly
    n = 9
    P = L.prolongation_1d(n).toarray()
    for I in range(5):
        for i in range(n):
            assert P[i, I] == pytest.approx(max(0.0, 1.0 - abs(i - 2 * I) / 2.0))


@pytest.mark.parametrize("co", [(True, True, False), (True, True, True), (False, True, True)])
def test_3d_galerkin_is_the_tensor_of_1d_galerkins(co):
    shape, W, alpha = (5, 6, 7), (1.0, 0.8, 0.1), 0.3
    for mass, stiff in ((L.mass_1d, L.stiff_1d), (L.identity_1d, L.fd_1d)):
        A = L.tensor_operator(shape, W, alpha, mass, stiff)
        Ac = L.galerkin(A, L.prolongation(shape, co)).toarray()
        nz, ny, nx = shape
        fac = []
        for n, c in zip((nx, ny, nz), co):
            p = L.prolongation_1d(n) if c else L.identity_1d(n)
            fac.append((L.galerkin(mass(n), p), L.galerkin(stiff(n), p)))
        (Mx, Kx), (My, Ky), (Mz, Kz) = fac
        T = (alpha * L.kron3(Mz, My, Mx) + W[0] * L.kron3(Mz, My, Kx) + W[1] * L.kron3(Mz, Ky, Mx)
             + W[2] * L.kron3(Kz, My, Mx)).toarray()
        np.testing.assert_allclose(Ac, T, atol=1e-13)
        # symmetric, PSD, coarse shape as stated
        np.testing.assert_allclose(Ac, Ac.T, atol=1e-14)
        assert np.linalg.eigvalsh(Ac).min() > -1e-10
        assert int(np.prod(L.coarse_shape(shape, co))) == Ac.shape[0]


def test_hybrid_fine_operator_is_the_constant_operator():
    # Hybrid keeps the 6-point Laplacian at the finest level
    shape, W, alpha = (3, 4, 5), (1.0, 1.0, 0.1), 0.2
    A = L.tensor_operator(shape, W, alpha, L.identity_1d, L.fd_1d)
    x = np.random.default_rng(5).random(shape)
    np.testing.assert_allclose((A @ x.ravel()).reshape(shape), O.apply_A(x, W, alpha), atol=1e-14)


# ---------------------------------------------------------------- solves
def test_linear_cg_equals_dense_solves():
    I0 = synth.make_stack(7, 6, 4, 0, "f32")
    I1 = L.diffuse_z_linear(I0)
    A = L.linear_operator(I0.shape, (1.0, 1.0, 0.1), 0.0).toarray()
    b = L.rhs_diffusion_linear(I0).ravel()
    N = A.shape[0]
    # bordered system pins the mean (reading L-3)
    Bd = np.zeros((N + 1, N + 1))
    Bd[:N, :N] = A
    Bd[:N, N] = Bd[N, :N] = 1.0
    rhs = np.concatenate([b, [O.decode(I0).sum()]])
    x = np.linalg.solve(Bd, rhs)[:N]
    np.testing.assert_allclose(I1.ravel(), x, atol=1e-9)
    I2 = L.screened_poisson_slices_linear(I0, I1, 0.01)
    A2 = L.linear_operator(I0.shape, (1.0, 1.0, 0.0), 0.01, per_slice=True).toarray()
    x2 = np.linalg.solve(A2, L.rhs_blend_linear(I0, I1, 0.01).ravel())
    np.testing.assert_allclose(I2.ravel(), x2, atol=1e-9)
    assert L.slice_rel_residuals_linear(I2, L.rhs_blend_linear(I0, I1, 0.01), 0.01).max() < 1e-9


def test_linear_invariants():
    rng = np.random.default_rng(6)
    c = np.full((4, 5, 6), 0.37)
    np.testing.assert_allclose(L.diffuse_z_linear(c), c, atol=1e-12)
    # z-invariant stack: G is the stack's own gradient, so it is the minimiser
    s = np.repeat(rng.random((1, 5, 6)), 4, axis=0)
    np.testing.assert_allclose(L.diffuse_z_linear(s), s, atol=1e-9)
    # identity blend: I1 = I0 gives I2 = I0 for any alpha
    J = rng.random((3, 5, 6))
    np.testing.assert_allclose(L.screened_poisson_slices_linear(J, J, 0.1), J, atol=1e-9)


def test_linear_differs_from_constant_but_agrees_on_smooth_data():
    # a different discrete answer on the rough synthetic stack (Table 1) ...
    I0 = synth.make_stack(16, 16, 6, 0, "f32")
    assert np.abs(L.diffuse_z_linear(I0) - O.diffuse_z(I0)).max() > 1e-3
    # ... of the same continuous problem: on a smooth field both discretisations agree to O(h^2)
    z, y, x = np.meshgrid(np.arange(6) / 5, np.arange(24) / 23, np.arange(24) / 23, indexing="ij")
    s = 0.5 + 0.2 * np.cos(np.pi * x) * np.cos(np.pi * y) + 0.1 * np.cos(np.pi * z) * np.cos(np.pi * x)
    d = np.abs(L.diffuse_z_linear(s) - O.diffuse_z(s)).max()
    assert d < 0.01, d
