"""CPU ORACLE (fp64, numpy / scipy.sparse) — TEST INFRASTRUCTURE ONLY; never imported by the product.

NEXT-3: the paper's other discretisations, PAPER.md:305-323 (§4.2).

* **Linear**: "the 26-point Laplacian stencil defined by using first-order B-splines as finite
  elements with the prolongation operator defined by the nesting of B-splines (using the stencil
  (1/2,1,1/2)^{(x)3})".  It changes the discrete answer, so the systems of the
  two phases are assembled here from their definition: the paper's energies (PAPER.md:148, 172,
  227) with I, I0, I1 replaced by their B-spline interpolants, minimised over the B-spline
  coefficients (Galerkin finite elements).
* **Hybrid**: "the 6-point Laplacian at the finest resolution but ... the prolongation operator
  for the first-order B-splines ... using the Galerkin formulation".  Its
  finest system is the Constant one (gdp_oracle.py), so its answer is gdp_oracle's; this module
  supplies the transfer and Galerkin operators both schemes use on the coarse levels.

Readings:
  L-1  one hat function per voxel, centred on the voxel centre, unit spacing; the energy is
       integrated over the hull of the voxel centres, [0, n-1] per axis (Neumann / natural
       boundary, as reading c-1 keeps only links inside the grid).  An axis with n = 1 has no
       extent and is not integrated over (mass 1, stiffness 0): one slice is a 2D problem.
  L-2  G = grad I0_h (x and y components) for phase 1; phase 2 per slice blends alpha I1_h with
       the gradients of I0_h.  Hence, with M / K the 1D mass / stiffness matrices and
       S_x = K (x) M (x) M etc. (z slowest):
         phase 1   (bx S_x + by S_y + bz S_z) I1 = (bx S_x + by S_y) I0         (alpha = 0)
         phase 2   (alpha M2 + S2) I2 = alpha M2 I1 + S2 I0   per slice, M2 = M (x) M.
  L-3  phase-1 null space (constants): the mean pin of c-3, mean(I1) = mean(I0) over voxels.
  L-4  transfers of Linear and Hybrid: coarse node I sits on fine node 2I, n_c = ceil(n/2);
       fine node 2I takes coarse I (weight 1), fine node 2I+1 takes 1/2 of I and 1/2 of I+1
       (the nesting hat(t/2) = 1/2 hat(t+1) + hat(t) + 1/2 hat(t-1)); on an even-length axis the
       last fine node 2I+1 has no coarse node I+1 and takes coarse I with weight 1, so that P
       reproduces constants (the Galerkin coarse operators keep the constant null space).
       Restriction R = P^T; coarse operators A_c = P^T A P (Galerkin).

Layout as gdp_oracle: numpy arrays (nz, ny, nx), x fastest; flat index z*ny*nx + y*nx + x.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .gdp_oracle import _as_f64, cg

# ---------------------------------------------------------------------------
# 1D element matrices of the hat basis on one element [0, 1] (reading L-1):
#   mass       int_0^1 phi_a phi_b dt    with phi_0 = 1 - t, phi_1 = t
#   stiffness  int_0^1 phi_a' phi_b' dt
# ---------------------------------------------------------------------------
ELEM_MASS = np.array([[1.0 / 3.0, 1.0 / 6.0], [1.0 / 6.0, 1.0 / 3.0]])
ELEM_STIFF = np.array([[1.0, -1.0], [-1.0, 1.0]])


def _assemble_1d(n: int, elem: np.ndarray, single: float) -> sp.csr_matrix:
    """Sum of the element matrices of the n-1 elements [i, i+1] of an axis of n nodes."""
    if n == 1:
        return sp.csr_matrix(np.array([[single]]))
    A = sp.lil_matrix((n, n))
    for e in range(n - 1):
        for a in range(2):
            for b in range(2):
                A[e + a, e + b] += elem[a, b]
    return A.tocsr()


def mass_1d(n: int) -> sp.csr_matrix:
    """M of reading L-1 (an axis of one node carries the unit point mass: no integration)."""
    return _assemble_1d(n, ELEM_MASS, 1.0)


def stiff_1d(n: int) -> sp.csr_matrix:
    """K of reading L-1 (0 on an axis of one node)."""
    return _assemble_1d(n, ELEM_STIFF, 0.0)


def identity_1d(n: int) -> sp.csr_matrix:
    return sp.identity(n, format="csr")


def fd_1d(n: int) -> sp.csr_matrix:
    """D^T D of the forward difference on the n-1 links of an axis (Constant / Hybrid fine level,
    reading c-2): the 1D block of gdp_oracle.apply_A."""
    if n == 1:
        return sp.csr_matrix((1, 1))
    D = sp.diags([-np.ones(n - 1), np.ones(n - 1)], [0, 1], shape=(n - 1, n))
    return (D.T @ D).tocsr()


def kron3(Az, Ay, Ax) -> sp.csr_matrix:
    """Az (x) Ay (x) Ax for the flat index z*ny*nx + y*nx + x."""
    return sp.kron(Az, sp.kron(Ay, Ax, format="csr"), format="csr")


# ---------------------------------------------------------------------------
# Operators of the two phases (reading L-2)
# ---------------------------------------------------------------------------
def tensor_operator(shape, W, alpha, mass=mass_1d, stiff=stiff_1d, per_slice=False) -> sp.csr_matrix:
    """alpha M(x)M(x)M + bx K(x)M(x)M + by M(x)K(x)M + bz M(x)M(x)K (axes in x, y, z order of W).

    per_slice: the z axis carries no coupling and no integration (independent 2D systems):
    its factor is the identity in every term and bz is ignored.
    """
    nz, ny, nx = shape
    Mx, My = mass(nx), mass(ny)
    Kx, Ky = stiff(nx), stiff(ny)
    if per_slice:
        Mz, Kz, bz = identity_1d(nz), None, 0.0
    else:
        Mz, Kz, bz = mass(nz), stiff(nz), W[2]
    A = alpha * kron3(Mz, My, Mx) + W[0] * kron3(Mz, My, Kx) + W[1] * kron3(Mz, Ky, Mx)
    if bz != 0.0:
        A = A + bz * kron3(Kz, My, Mx)
    return A.tocsr()


def linear_operator(shape, W, alpha, per_slice=False) -> sp.csr_matrix:
    """The Linear finite-element matrix of the §4 operator (alpha - div W grad)."""
    return tensor_operator(shape, W, alpha, per_slice=per_slice)


def apply_factors(u, fx, fy, fz) -> np.ndarray:
    """(fz (x) fy (x) fx) u applied one axis at a time (fx first, so that a stiffness factor sees
    the data before any mass sum: the gradient terms of a constant are exactly 0)."""
    u = np.asarray(u, dtype=np.float64)
    for f, ax in ((fx, 2), (fy, 1), (fz, 0)):
        if f is not None:
            u = np.moveaxis(np.tensordot(f.toarray(), u, axes=([1], [ax])), 0, ax)
    return u


def rhs_diffusion_linear(I0, W=(1.0, 1.0, 0.1)) -> np.ndarray:
    """Phase 1 rhs (reading L-2): (bx S_x + by S_y) I0 — the z component of G is 0."""
    I = _as_f64(I0)
    nz, ny, nx = I.shape
    Sx = apply_factors(I, stiff_1d(nx), mass_1d(ny), mass_1d(nz))
    Sy = apply_factors(I, None, stiff_1d(ny), None)
    Sy = apply_factors(Sy, mass_1d(nx), None, mass_1d(nz))
    return W[0] * Sx + W[1] * Sy


def rhs_blend_linear(I0, I1, alpha) -> np.ndarray:
    """Phase 2 rhs per slice (reading L-2): alpha M2 I1 + S2 I0."""
    I = _as_f64(I0)
    J = np.asarray(I1, dtype=np.float64)
    nz, ny, nx = I.shape
    M2 = apply_factors(J, mass_1d(nx), mass_1d(ny), None)
    Sx = apply_factors(I, stiff_1d(nx), mass_1d(ny), None)
    Sy = apply_factors(apply_factors(I, None, stiff_1d(ny), None), mass_1d(nx), None, None)
    return alpha * M2 + Sx + Sy


def apply_linear(x, W, alpha, per_slice=False) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    return (linear_operator(x.shape, W, alpha, per_slice) @ x.ravel()).reshape(x.shape)


def diffuse_z_linear(I0, W=(1.0, 1.0, 0.1), tol=1e-10, return_info=False):
    """Phase 1 under Linear: CG from x0 = I0, then the mean pin (reading L-3)."""
    I = _as_f64(I0)
    A = linear_operator(I.shape, W, 0.0)
    b = rhs_diffusion_linear(I, W)
    b = b - b.mean()  # 1^T b = 0 exactly (K 1 = 0); removes rounding only
    if np.abs(b).max() <= 1e-13 * max(1.0, np.abs(I).max()):
        # no x / y gradients (e.g. a constant stack): b is 0 up to the rounding of its sums, the
        # minimiser is a constant and the mean pin makes it mean(I0); CG relative to a rounding-
        # level ||b|| would chase that rounding instead
        I1 = np.full(I.shape, I.mean())
        return (I1, {"iterations": 0, "rel_res": 0.0}) if return_info else I1
    x, info = cg(lambda u: (A @ u.ravel()).reshape(u.shape), b, I, tol=tol)
    I1 = x + (I.mean() - x.mean())
    return (I1, info) if return_info else I1


def screened_poisson_slices_linear(I0, I1, alpha=0.01, tol=1e-10, return_info=False):
    """Phase 2 under Linear: per-slice CG from x0 = I0 with per-slice stopping."""
    if not alpha > 0:
        raise ValueError("screened Poisson needs alpha > 0")
    I = _as_f64(I0)
    A = linear_operator(I.shape, (1.0, 1.0, 0.0), alpha, per_slice=True)
    b = rhs_blend_linear(I, I1, alpha)
    x, info = cg(lambda u: (A @ u.ravel()).reshape(u.shape), b, I, tol=tol, axes=(1, 2))
    return (x, info) if return_info else x


def destripe_linear(I0, alpha=0.01, W=(1.0, 1.0, 0.1), tol=1e-10):
    I1 = diffuse_z_linear(I0, W, tol)
    return I1, screened_poisson_slices_linear(I0, I1, alpha, tol)


def slice_rel_residuals_linear(x, b, alpha) -> np.ndarray:
    """Per-slice ||b_i - A x_i|| / ||b_i|| of the Linear phase-2 systems."""
    r = np.asarray(b, dtype=np.float64) - apply_linear(x, (1.0, 1.0, 0.0), alpha, per_slice=True)
    b = np.asarray(b, dtype=np.float64)
    return np.sqrt((r * r).sum(axis=(1, 2))) / np.sqrt((b * b).sum(axis=(1, 2)))


def rel_residual_linear(x, b, W, alpha, per_slice=False) -> float:
    r = np.asarray(b, dtype=np.float64) - apply_linear(x, W, alpha, per_slice)
    return float(np.linalg.norm(r.ravel()) / np.linalg.norm(np.asarray(b, dtype=np.float64).ravel()))


# ---------------------------------------------------------------------------
# Transfers and Galerkin coarse operators (reading L-4)
# ---------------------------------------------------------------------------
def prolongation_1d(n: int) -> sp.csr_matrix:
    """P (n x ceil(n/2)) of reading L-4, written node by node."""
    nc = (n + 1) // 2
    P = sp.lil_matrix((n, nc))
    for i in range(n):
        I = i // 2
        if i % 2 == 0:
            P[i, I] = 1.0
        elif I + 1 < nc:
            P[i, I] = 0.5
            P[i, I + 1] = 0.5
        else:
            P[i, I] = 1.0
    return P.tocsr()


def prolongation(shape, coarsen) -> sp.csr_matrix:
    """3D P = Pz (x) Py (x) Px; an axis that is not coarsened (coarsen[d] False, d in x, y, z
    order) keeps the identity."""
    nz, ny, nx = shape
    f = [prolongation_1d(n) if c else identity_1d(n) for n, c in zip((nx, ny, nz), coarsen)]
    return kron3(f[2], f[1], f[0])


def coarse_shape(shape, coarsen):
    nz, ny, nx = shape
    c = [((n + 1) // 2 if k else n) for n, k in zip((nx, ny, nz), coarsen)]
    return (c[2], c[1], c[0])


def galerkin(A: sp.spmatrix, P: sp.spmatrix) -> sp.csr_matrix:
    """A_c = P^T A P ("the Galerkin formulation")."""
    return (P.T @ A @ P).tocsr()


def hierarchy(shape, A: sp.spmatrix, coarsenings):
    """Fine-to-coarse list of (shape, A_l) for the given per-level coarsening flags."""
    out = [(tuple(shape), A.tocsr())]
    for co in coarsenings:
        s, Al = out[-1]
        P = prolongation(s, co)
        out.append((coarse_shape(s, co), galerkin(Al, P)))
    return out
