"""CLOSED-FORM CPU ORACLE (fp64, scipy DCT-II) — TEST INFRASTRUCTURE ONLY.

PAPER.md §3.2 (lines 186-218) interprets both phases in frequency space:
  AD  (§3.2.1): I1_klm = (bx k^2 + by l^2) / (bx k^2 + by l^2 + bz m^2) * I0_klm
                (the garbled "beta_z^2 m^2" of PAPER.md:195 is read as beta_z m^2, c-4)
  SP  (§3.2.2): I2_klm = (alpha I1_klm + (k^2 + l^2) I0_klm) / (alpha + k^2 + l^2)
The paper states them for complex exponentials (periodic, continuous symbol k^2).
On the Neumann grid of reading c-1 the same statements hold exactly with the
cosine (DCT-II) eigenbasis of the path-graph Laplacian L_n = D^T D, whose
eigenvalue for mode k is  mu_k = 4 sin^2(pi k / (2 n))  (the discrete k^2).
This module is that discrete analog: an O(N log N) exact solve usable at the
full config sizes where CG is infeasible.
"""
from __future__ import annotations

import numpy as np
import scipy.fft as sfft


def path_eigenvalues(n: int) -> np.ndarray:
    """mu_k = 4 sin^2(pi k / 2n), k = 0..n-1: the spectrum of L_n = D^T D (Neumann path graph)."""
    k = np.arange(n, dtype=np.float64)
    return 4.0 * np.sin(np.pi * k / (2.0 * n)) ** 2


def _mu3(shape):
    nz, ny, nx = shape
    return (path_eigenvalues(nx)[None, None, :], path_eigenvalues(ny)[None, :, None],
            path_eigenvalues(nz)[:, None, None])


def _dct(a, axes, workers):
    return sfft.dctn(a, type=2, norm="ortho", axes=axes, workers=workers)


def _idct(a, axes, workers):
    return sfft.idctn(a, type=2, norm="ortho", axes=axes, workers=workers)


def _as_f64(I0):
    I0 = np.asarray(I0)
    if I0.dtype == np.uint8:
        return (I0.astype(np.float32) / np.float32(255.0)).astype(np.float64)
    return I0.astype(np.float64)


def ad_gain(mx, my, mz, W=(1.0, 1.0, 0.1)):
    """§3.2.1 gain with discrete symbols; the DC mode (0,0,0) has gain 1 (mean pin, c-3)."""
    num = W[0] * mx + W[1] * my
    den = num + W[2] * mz
    with np.errstate(invalid="ignore", divide="ignore"):
        g = np.where(den > 0, num / np.where(den > 0, den, 1.0), 1.0)
    return g


def sp_gain(mx, my, alpha):
    """§3.2.2 gain of an I1-only mode alpha/(alpha + mu_kl) (the I0 term gets mu/(alpha+mu))."""
    return alpha / (alpha + mx + my)


def combined_gain(mx, my, mz, alpha, W=(1.0, 1.0, 0.1)):
    """§3.2.3 F_klm = (alpha g_AD + mu_kl) / (alpha + mu_kl) with discrete symbols."""
    mu = mx + my
    return (alpha * ad_gain(mx, my, mz, W) + mu) / (alpha + mu)


def diffuse_z_dct(I0, W=(1.0, 1.0, 0.1), workers=-1):
    """Phase 1 by §3.2.1 in the DCT-II basis of the Neumann grid. Returns fp64 I1."""
    I = _as_f64(I0)
    mx, my, mz = _mu3(I.shape)
    Ih = _dct(I, (0, 1, 2), workers)
    Ih *= ad_gain(mx, my, mz, W)
    return _idct(Ih, (0, 1, 2), workers)


def screened_poisson_slices_dct(I0, I1, alpha=0.01, workers=-1):
    """Phase 2 by §3.2.2, per slice (2D DCT-II over x, y). Returns fp64 I2."""
    I = _as_f64(I0)
    J = np.asarray(I1, dtype=np.float64)
    mx, my, _ = _mu3(I.shape)
    mu = mx + my
    Ih = _dct(I, (1, 2), workers)
    Jh = _dct(J, (1, 2), workers)
    out = (alpha * Jh + mu * Ih) / (alpha + mu)
    del Ih, Jh
    return _idct(out, (1, 2), workers)


def dct_solve(b, W, alpha, mean=0.0, workers=-1):
    """Exact solve of (alpha + sum_d beta_d L_d) x = b on the Neumann grid.

    Coupled axes are those with beta_d > 0; uncoupled axes are independent systems.
    If alpha == 0 the constant mode of each system is set so that its mean is `mean`.
    """
    b = np.asarray(b, dtype=np.float64)
    axes = tuple(ax for ax, w in zip((2, 1, 0), W) if w > 0 and b.shape[ax] > 1)
    mx, my, mz = _mu3(b.shape)
    lam = alpha + (W[0] * mx if 2 in axes else 0.0) + (W[1] * my if 1 in axes else 0.0) \
        + (W[2] * mz if 0 in axes else 0.0)
    lam = np.broadcast_to(lam, b.shape) if np.ndim(lam) else np.full(b.shape, lam)
    bh = _dct(b, axes, workers) if axes else b.copy()
    xh = np.where(lam > 0, bh / np.where(lam > 0, lam, 1.0), 0.0)
    x = _idct(xh, axes, workers) if axes else xh
    if alpha == 0.0 and axes:
        x = x - x.mean(axis=axes, keepdims=True) + mean
    return x
