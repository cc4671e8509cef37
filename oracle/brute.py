"""BRUTE-FORCE ENERGY ORACLE (pure Python, tiny grids) — TEST INFRASTRUCTURE ONLY.

Pins the assembled operator and right-hand sides of `gdp_oracle` to the energies
the paper minimises, evaluated voxel by voxel and link by link:

  §4:   E(I) = sum_voxels alpha (I - V)^2
                                  + sum_links beta_d ((I_n - I_c) - G_link)^2
  §3.1.1: alpha = 0, G = (dI0/dx, dI0/dy, 0), W = Diag(bx, by, bz)
  §3.1.2: per slice, alpha (I - I1)^2 + |grad I - grad I0|^2

E is quadratic, E(I) = I^T A I - 2 b^T I + c, so A and b are recovered exactly by
polarisation (A_ij = (E(e_i + e_j) - E(e_i) - E(e_j) + E(0)) / 2, b_i = (E(-e_i) - E(e_i)) / 4),
with no use of the oracle's difference/transpose routines.  Grids of <= ~100 voxels.
"""
from __future__ import annotations

import itertools

import numpy as np


def _links(shape):
    """All (c, n, axis) links between face-adjacent voxels inside the grid (reading c-1)."""
    nz, ny, nx = shape
    out = []
    for z, y, x in itertools.product(range(nz), range(ny), range(nx)):
        if x + 1 < nx:
            out.append(((z, y, x), (z, y, x + 1), 0))
        if y + 1 < ny:
            out.append(((z, y, x), (z, y + 1, x), 1))
        if z + 1 < nz:
            out.append(((z, y, x), (z + 1, y, x), 2))
    return out


def energy(I, shape, W, alpha, V=None, G=None):
    """E(I) of §4 as plain sums. G maps a link (c, n, axis) to its target difference."""
    links = _links(shape)
    e = 0.0
    if alpha:
        for idx in itertools.product(*(range(s) for s in shape)):
            v = 0.0 if V is None else V[idx]
            e += alpha * (I[idx] - v) ** 2
    for c, n, ax in links:
        g = 0.0 if G is None else G(c, n, ax)
        e += W[ax] * ((I[n] - I[c]) - g) ** 2
    return e


def quadratic_form(shape, W, alpha, V=None, G=None):
    """Recover (A, b) of E(I) = I^T A I - 2 b^T I + c by polarisation."""
    N = int(np.prod(shape))

    def E(vec):
        return energy(vec.reshape(shape), shape, W, alpha, V, G)

    zero = np.zeros(N)
    E0 = E(zero)
    Ee = np.empty(N)
    Em = np.empty(N)
    for i in range(N):
        e = zero.copy()
        e[i] = 1.0
        Ee[i] = E(e)
        Em[i] = E(-e)
    b = (Em - Ee) / 4.0
    # quadratic part Q(e_i) = (E(e_i) + E(-e_i))/2 - E0
    Q = (Ee + Em) / 2.0 - E0
    A = np.diag(Q)
    for i in range(N):
        for j in range(i + 1, N):
            e = zero.copy()
            e[i] = 1.0
            e[j] = 1.0
            Qij = (E(e) + E(-e)) / 2.0 - E0
            A[i, j] = A[j, i] = (Qij - Q[i] - Q[j]) / 2.0
    return A, b


def diffusion_G(I0):
    """Target gradient of §3.1.1: G = (dI0/dx, dI0/dy, 0) on each link."""
    def G(c, n, ax):
        return 0.0 if ax == 2 else float(I0[n] - I0[c])
    return G


def minimiser(A, b, singular_mean=None):
    """Dense minimiser of E: A x = b (least squares + mean pin when A is singular)."""
    if singular_mean is None:
        return np.linalg.solve(A, b)
    x = np.linalg.lstsq(A, b, rcond=None)[0]
    return x - x.mean() + singular_mean


def npr_G(I0, lam, sigma):
    """Target gradient of the §6 NPR filter link by link: the gradient
    magnitude is the 3D forward-difference gradient at the link's base voxel (reading n-1)."""
    shape = I0.shape

    def mag2(c):
        z, y, x = c
        s = 0.0
        for dz, dy, dx in ((0, 0, 1), (0, 1, 0), (1, 0, 0)):
            n = (z + dz, y + dy, x + dx)
            if n[0] < shape[0] and n[1] < shape[1] and n[2] < shape[2]:
                s += float(I0[n] - I0[c]) ** 2
        return s

    def G(c, n, ax):
        return lam * (1.0 - np.exp(-mag2(c) / (2.0 * sigma * sigma))) * float(I0[n] - I0[c])
    return G
