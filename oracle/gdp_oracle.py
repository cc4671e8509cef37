"""CPU ORACLE (fp64, numpy) — TEST INFRASTRUCTURE ONLY; never imported by the product.

Plain definition of what the hot path computes:
assemble the paper's discrete operators with Neumann boundaries and solve the
linear systems by textbook conjugate gradient to ||b - A x|| <= 1e-10 ||b||.

Arrays are numpy, shape (nz, ny, nx) — slice-major, x fastest.
Axis 2 is x, axis 1 is y, axis 0 is z.  Weights W = (beta_x, beta_y, beta_z).

Readings of the paper used here:
  c-1  boundary condition: Neumann = links exist only between two voxels of the grid.
  c-2  discrete gradient = forward difference on links (D); divergence = -D^T.
  c-3  alpha = 0 diffusion is singular; rhs is projected to mean 0 and the
       solution is pinned so that mean(I1) = mean(I0).
  c-5  the AD energy is (grad I - G)^T W (grad I - G) (stray transpose dropped).
  c-7  residual measure ||b - A x||_2 / ||b||_2 with b the phase's finest rhs;
       phase 2 is one system per slice.
  c-9  u8 input decodes to u8/255 rounded to fp32 (the exact values the GPU sees).
  c-10 no output clipping.
"""
from __future__ import annotations

import numpy as np

AXIS = {"x": 2, "y": 1, "z": 0}


# ---------------------------------------------------------------------------
# a1: input decode — PAPER.md:143-144 (I^0 is the input voxel data); reading c-9
# ---------------------------------------------------------------------------
def decode(I0: np.ndarray) -> np.ndarray:
    """fp64 copy of the fp32 values the GPU consumes: u8/255 rounded to fp32, or fp32 as is."""
    I0 = np.asarray(I0)
    if I0.dtype == np.uint8:
        return (I0.astype(np.float32) / np.float32(255.0)).astype(np.float64)
    return I0.astype(np.float32).astype(np.float64)


def _as_f64(I0) -> np.ndarray:
    """u8 / fp32 inputs go through `decode`; fp64 inputs (analytic test fields) stay exact."""
    I0 = np.asarray(I0)
    return I0 if I0.dtype == np.float64 else decode(I0)


# ---------------------------------------------------------------------------
# Discrete gradient / divergence on links — reading c-1, c-2
# ---------------------------------------------------------------------------
def forward_difference(u: np.ndarray, axis: int) -> np.ndarray:
    """D_d u: the (n_d - 1) link values u[i+1] - u[i] along `axis` (no link leaves the grid)."""
    return np.diff(u, axis=axis)


def forward_difference_T(g: np.ndarray, axis: int) -> np.ndarray:
    """D_d^T g for a link field g: (D^T g)[i] = g[i-1] - g[i], absent links count as 0."""
    pad = [(0, 0)] * g.ndim
    pad[axis] = (1, 1)
    gp = np.pad(g, pad)
    lo = [slice(None)] * g.ndim
    hi = [slice(None)] * g.ndim
    lo[axis] = slice(0, -1)
    hi[axis] = slice(1, None)
    return gp[tuple(lo)] - gp[tuple(hi)]


def gradient(I: np.ndarray, axes=("x", "y", "z")) -> dict:
    """nabla I as link fields {axis: D_axis I} (PAPER.md:145 uses d/dx, d/dy on slices)."""
    return {a: forward_difference(I, AXIS[a]) for a in axes}


def divergence(F: dict, W=(1.0, 1.0, 1.0)) -> np.ndarray:
    """nabla . (W F) = -sum_d beta_d D_d^T F_d  (reading c-2)."""
    beta = {"x": W[0], "y": W[1], "z": W[2]}
    out = None
    for a, g in F.items():
        t = -beta[a] * forward_difference_T(g, AXIS[a])
        out = t if out is None else out + t
    return out


# ---------------------------------------------------------------------------
# Operator of §4: (alpha - nabla . W nabla)  — PAPER.md:223-232
# ---------------------------------------------------------------------------
def apply_A(x: np.ndarray, W, alpha: float) -> np.ndarray:
    """A x = alpha x - nabla.(W nabla x) = alpha x + sum_d beta_d D_d^T D_d x."""
    x = np.asarray(x, dtype=np.float64)
    out = alpha * x
    for a, d in (("x", 0), ("y", 1), ("z", 2)):
        if W[d] != 0.0 and x.shape[AXIS[a]] > 1:
            out = out + W[d] * forward_difference_T(forward_difference(x, AXIS[a]), AXIS[a])
    return out


def rhs_general(V, G: dict, W, alpha: float) -> np.ndarray:
    """b = alpha V - nabla.(W G)  (the rhs of the general system of §4)."""
    b = -divergence(G, W) if G else 0.0
    if alpha != 0.0:
        b = b + alpha * np.asarray(V, dtype=np.float64)
    return np.asarray(b, dtype=np.float64)


def rhs_diffusion(I0f: np.ndarray, W=(1.0, 1.0, 0.1)) -> np.ndarray:
    """Eq. (1): Delta_W I1 = nabla.(W G) with G = (dI0/dx, dI0/dy, 0).

    Written as the §4 system with alpha = 0: (-nabla.W nabla) I1 = -nabla.(W G).
    """
    G = gradient(I0f, axes=("x", "y"))  # the z component of G is 0
    return rhs_general(None, G, W, 0.0)


def rhs_blend(I0f: np.ndarray, I1f: np.ndarray, alpha: float) -> np.ndarray:
    """Eq. (2): (alpha - Delta_pi) I2 = alpha I1 - Delta_pi I0, pi = Diag(1,1,0)."""
    G = gradient(I0f, axes=("x", "y"))
    return rhs_general(np.asarray(I1f, dtype=np.float64), G, (1.0, 1.0, 0.0), alpha)


# ---------------------------------------------------------------------------
# Textbook conjugate gradient (fp64).  `axes=None`: one system; axes=(1,2):
# independent per-slice systems with their own scalars and stopping tests.
# ---------------------------------------------------------------------------
def cg(applyA, b, x0, tol=1e-10, maxiter=200000, axes=None, restarts=5):
    b = np.asarray(b, dtype=np.float64)
    x = np.array(x0, dtype=np.float64, copy=True)

    def dot(u, v):
        return np.sum(u * v, axis=axes, keepdims=axes is not None)

    bb = dot(b, b)
    r0 = b - applyA(x)
    # relative to ||b||; a zero rhs (compatible singular case) is measured against ||r0||
    thr = (tol * tol) * np.where(bb > 0, bb, dot(r0, r0))
    total = 0
    for _ in range(restarts + 1):
        r = b - applyA(x)
        rr = dot(r, r)
        active = rr > thr
        if not np.any(active):
            break
        p = r.copy()
        it = 0
        while np.any(active) and it < maxiter:
            Ap = applyA(p)
            pAp = dot(p, Ap)
            active = active & (pAp > 0)
            a = np.where(active, rr / np.where(pAp > 0, pAp, 1.0), 0.0)
            x += a * p
            r -= a * Ap
            rr_new = dot(r, r)
            beta = np.where(active, rr_new / np.where(rr > 0, rr, 1.0), 0.0)
            p = r + beta * p
            rr = rr_new
            active = rr > thr
            it += 1
        total += it
    r = b - applyA(x)
    rel = np.sqrt(dot(r, r) / np.where(bb > 0, bb, 1.0))
    return x, {"iterations": total, "rel_res": rel}


# ---------------------------------------------------------------------------
# The two phases
# ---------------------------------------------------------------------------
def diffuse_z(I0, W=(1.0, 1.0, 0.1), tol=1e-10, return_info=False):
    """Phase 1, Eq. (1): I1 minimising the AD energy.

    alpha = 0 is singular (constants); b is projected to mean 0 (it is 0 up to
    rounding, 1^T D^T = 0) and I1 is pinned so that mean(I1) = mean(I0) (c-3).
    CG starts from x0 = I0.
    """
    I = _as_f64(I0)
    b = rhs_diffusion(I, W)
    b = b - b.mean()
    x, info = cg(lambda u: apply_A(u, W, 0.0), b, I, tol=tol)
    I1 = x + (I.mean() - x.mean())
    return (I1, info) if return_info else I1


def screened_poisson_slices(I0, I1, alpha=0.01, tol=1e-10, return_info=False):
    """Phase 2, Eq. (2): per slice (alpha - Delta) I2_i = alpha I1_i - Delta I0_i.

    alpha > 0: each slice system is SPD; CG per slice from x0 = I0, per-slice stopping.
    """
    if not alpha > 0:
        raise ValueError("screened Poisson needs alpha > 0")
    I = _as_f64(I0)
    b = rhs_blend(I, I1, alpha)
    x, info = cg(lambda u: apply_A(u, (1.0, 1.0, 0.0), alpha), b, I, tol=tol, axes=(1, 2))
    return (x, info) if return_info else x


def destripe(I0, alpha=0.01, W=(1.0, 1.0, 0.1), tol=1e-10):
    """Both phases: I2 = SP(I0, AD(I0))."""
    I1 = diffuse_z(I0, W, tol)
    return I1, screened_poisson_slices(I0, I1, alpha, tol)


# ---------------------------------------------------------------------------
# Residual measure (reading c-7)
# ---------------------------------------------------------------------------
def residual(x, b, W, alpha) -> np.ndarray:
    return np.asarray(b, dtype=np.float64) - apply_A(np.asarray(x, dtype=np.float64), W, alpha)


def rel_residual(x, b, W, alpha) -> float:
    r = residual(x, b, W, alpha)
    bn = np.linalg.norm(np.asarray(b, dtype=np.float64).ravel())
    return float(np.linalg.norm(r.ravel()) / bn) if bn > 0 else float(np.linalg.norm(r.ravel()))


def slice_rel_residuals(x, b, alpha) -> np.ndarray:
    """Per-slice ||b_i - A x_i|| / ||b_i|| for the phase-2 systems (W = pi)."""
    r = residual(x, b, (1.0, 1.0, 0.0), alpha)
    b = np.asarray(b, dtype=np.float64)
    rn = np.sqrt(np.sum(r * r, axis=(1, 2)))
    bn = np.sqrt(np.sum(b * b, axis=(1, 2)))
    return rn / np.where(bn > 0, bn, 1.0)


# ---------------------------------------------------------------------------
# NEXT-1: the §6 NPR filter (after Bhat et al. §6.2)
#   I1 = argmin  alpha (I - I0)^2 + || grad I - V ||_W^2,
#   V  = lam (1 - exp(-|grad I0|^2 / (2 sigma^2))) grad I0
# Readings: n-1 |grad I0|^2 of a link is the squared norm of the full 3D
# forward-difference gradient at the link's base voxel (absent links contribute 0);
# n-2 sigma = 5 on the paper's [0,256) gray scale is 5/255 on the u8/255 scale used here (c-9).
# ---------------------------------------------------------------------------
def npr_gradient_field(I0f, lam: float, sigma: float) -> dict:
    """V_{lam,sigma} on links {axis: values of the (n_d - 1) links}."""
    I = np.asarray(I0f, dtype=np.float64)
    G = gradient(I)
    mag2 = np.zeros(I.shape)
    for a, g in G.items():
        pad = [(0, 0)] * I.ndim
        pad[AXIS[a]] = (0, 1)  # the last voxel along the axis has no forward link
        mag2 += np.pad(g, pad) ** 2
    V = {}
    for a, g in G.items():
        base = [slice(None)] * I.ndim
        base[AXIS[a]] = slice(0, -1)  # link (c, c + e_a) has base voxel c
        V[a] = lam * (1.0 - np.exp(-mag2[tuple(base)] / (2.0 * sigma * sigma))) * g
    return V


def rhs_npr(I0f, W, alpha, lam, sigma) -> np.ndarray:
    """b = alpha I0 - nabla.(W V)  (the §4 rhs with V as the gradient target)."""
    I = np.asarray(I0f, dtype=np.float64)
    return rhs_general(I, npr_gradient_field(I, lam, sigma), W, alpha)


def npr_filter(I0, W=(1.0, 1.0, 0.1), alpha=0.001, lam=1.25, sigma=5.0 / 255.0, tol=1e-10, return_info=False):
    """§6 NPR filter: (alpha - nabla.W nabla) I1 = alpha I0 - nabla.(W V), CG from x0 = I0."""
    if not alpha > 0:
        raise ValueError("the NPR filter is a screened solve (alpha > 0)")
    I = _as_f64(I0)
    b = rhs_npr(I, W, alpha, lam, sigma)
    x, info = cg(lambda u: apply_A(u, W, alpha), b, I, tol=tol)
    return (x, info) if return_info else x
