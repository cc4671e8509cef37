"""Design prototype (numpy, fp32) of the GPU multigrid — NOT the oracle, NOT the product.

Used once to choose the coarsening rule, transfers, smoother sweeps and the
coarsest-level size before writing CUDA; imports neither oracle/ nor the package.
Run: python tools/mg_proto.py
"""
import sys

import numpy as np
import scipy.fft as sfft

F = np.float32


def stencil_apply(x, W, alpha):
    """alpha x + sum_d beta_d sum_{valid nbrs} (x_c - x_n), difference form (fp32)."""
    out = F(alpha) * x
    for ax, beta in ((2, W[0]), (1, W[1]), (0, W[2])):
        if beta == 0 or x.shape[ax] == 1:
            continue
        d = np.diff(x, axis=ax)  # x[i+1]-x[i]
        pad = [(0, 0)] * 3
        pad[ax] = (1, 1)
        dp = np.pad(d, pad)
        sl_lo = [slice(None)] * 3
        sl_hi = [slice(None)] * 3
        sl_lo[ax] = slice(0, -1)
        sl_hi[ax] = slice(1, None)
        out = out + F(beta) * (dp[tuple(sl_lo)] - dp[tuple(sl_hi)])
    return out


def diag(shape, W, alpha):
    D = np.full(shape, alpha, np.float32)
    for ax, beta in ((2, W[0]), (1, W[1]), (0, W[2])):
        n = shape[ax]
        if beta == 0 or n == 1:
            continue
        cnt = np.full(n, 2.0, np.float32)
        cnt[0] = cnt[-1] = 1.0
        sh = [1, 1, 1]
        sh[ax] = n
        D = D + F(beta) * cnt.reshape(sh)
    return D


def rb_sweep(x, b, W, alpha, D, color_masks, nsweeps):
    for _ in range(nsweeps):
        for m in color_masks:
            r = b - stencil_apply(x, W, alpha)
            x[m] += r[m] / D[m]
    return x


def R1(nf, nc):
    """Full weighting (1,3,3,1)/8 per axis, reflect at boundary, row-normalised."""
    P = P1(nf, nc)
    R = P.T.copy()
    R /= R.sum(axis=1, keepdims=True)
    return R


def P1(nf, nc):
    P = np.zeros((nf, nc), np.float64)
    for i in range(nf):
        I = i // 2
        J = I - 1 if i % 2 == 0 else I + 1
        if J < 0 or J >= nc:
            J = I
        P[i, I] += 0.75
        P[i, J] += 0.25
    return P


def apply_sep(x, mats):
    """mats = (Mz, My, Mx) or None per axis."""
    out = x.astype(np.float64)
    for ax, M in zip((0, 1, 2), mats):
        if M is not None:
            out = np.moveaxis(np.tensordot(M, np.moveaxis(out, ax, 0), axes=(1, 0)), 0, ax)
    return out.astype(np.float32)


def build_levels(shape, W, alpha, coarse_max=4096, dim_max=64):
    levels = [dict(shape=shape, W=tuple(W), alpha=alpha)]
    while True:
        L = levels[-1]
        nz, ny, nx = L["shape"]
        n = {2: nx, 1: ny, 0: nz}
        Wd = {2: L["W"][0], 1: L["W"][1], 0: L["W"][2]}
        coupled = [ax for ax in (2, 1, 0) if Wd[ax] > 0 and n[ax] > 1]
        size = int(np.prod([n[a] for a in coupled])) if coupled else 1
        if not coupled or (size <= coarse_max and max(n[a] for a in coupled) <= dim_max):
            break
        wmax = max(Wd[a] for a in coupled)
        co = [a for a in coupled if Wd[a] >= 0.5 * wmax]
        new = dict(n)
        Wn = dict(Wd)
        for a in co:
            new[a] = (n[a] + 1) // 2
            Wn[a] = Wd[a] / 4.0
        levels.append(dict(shape=(new[0], new[1], new[2]), W=(Wn[2], Wn[1], Wn[0]), alpha=alpha,
                           coarsened=co))
    return levels


def coarse_solve(b, W, alpha):
    b = b.astype(np.float64)
    axes = tuple(ax for ax, w in zip((2, 1, 0), W) if w > 0 and b.shape[ax] > 1)
    mu = [4 * np.sin(np.pi * np.arange(n) / (2 * n)) ** 2 for n in b.shape]
    lam = alpha + 0.0 * b
    for ax, w in zip((2, 1, 0), W):
        if ax in axes:
            sh = [1, 1, 1]
            sh[ax] = b.shape[ax]
            lam = lam + w * mu[ax].reshape(sh)
    bh = sfft.dctn(b, type=2, norm="ortho", axes=axes) if axes else b
    xh = np.where(lam > 0, bh / np.where(lam > 0, lam, 1), 0)
    x = sfft.idctn(xh, type=2, norm="ortho", axes=axes) if axes else xh
    return x.astype(np.float32)


def vcycle(levels, x0, b0, nu1, nu2, masks, diags, mats):
    xs = [x0] + [None] * (len(levels) - 1)
    bs = [b0] + [None] * (len(levels) - 1)
    for l in range(len(levels) - 1):
        L = levels[l]
        if l > 0:
            xs[l] = np.zeros(L["shape"], np.float32)
        rb_sweep(xs[l], bs[l], L["W"], L["alpha"], diags[l], masks[l], nu1)
        r = bs[l] - stencil_apply(xs[l], L["W"], L["alpha"])
        bs[l + 1] = apply_sep(r, mats[l + 1][0])
    Lc = levels[-1]
    xs[-1] = coarse_solve(bs[-1], Lc["W"], Lc["alpha"])
    for l in range(len(levels) - 2, -1, -1):
        L = levels[l]
        xs[l] += apply_sep(xs[l + 1], mats[l + 1][1])
        rb_sweep(xs[l], bs[l], L["W"], L["alpha"], diags[l], masks[l], nu2)
    return xs[0]


def prepare(levels):
    masks, diags, mats = [], [], [None]
    for l, L in enumerate(levels):
        nz, ny, nx = L["shape"]
        z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        par = (x + y + z) % 2
        masks.append([par == 0, par == 1])
        diags.append(diag(L["shape"], L["W"], L["alpha"]))
        if l > 0:
            f = levels[l - 1]["shape"]
            c = L["shape"]
            Rm = tuple(R1(f[a], c[a]) if f[a] != c[a] else None for a in (0, 1, 2))
            Pm = tuple(P1(f[a], c[a]) if f[a] != c[a] else None for a in (0, 1, 2))
            mats.append((Rm, Pm))
    return masks, diags, mats


def run(I0, phase, alpha=0.01, nu1=2, nu2=2, ncyc=8, I1=None):
    I0 = I0.astype(np.float32)
    if phase == 1:
        W = (1.0, 1.0, 0.1)
        b = stencil_apply(I0, (1.0, 1.0, 0.0), 0.0)
        al = 0.0
    else:
        W = (1.0, 1.0, 0.0)
        al = alpha
        b = F(alpha) * I1.astype(np.float32) + stencil_apply(I0, (1.0, 1.0, 0.0), 0.0)
    levels = build_levels(I0.shape, W, al)
    print("levels:", [L["shape"] for L in levels])
    masks, diags, mats = prepare(levels)
    x = I0.copy()
    b64 = b.astype(np.float64)
    bn = np.linalg.norm(b64)
    hist = []
    for k in range(ncyc):
        x = vcycle(levels, x, b, nu1, nu2, masks, diags, mats)
        r = b64 - stencil_apply(x.astype(np.float64), W, al)  # fp64 eval
        hist.append(np.linalg.norm(r) / bn)
    return x, hist


if __name__ == "__main__":
    sys.path.insert(0, ".")
    import gdp_synth as g
    for shape in [(16, 64, 64), (32, 128, 128), (33, 97, 75), (128, 64, 64)]:
        nz, ny, nx = shape
        I0 = g.make_stack(nx, ny, nz, 0, "f32")
        for nu in (1, 2):
            x, h = run(I0, 1, nu1=nu, nu2=nu)
            print(shape, "AD nu", nu, " ".join(f"{v:.1e}" for v in h))
        I1 = x
        for a in (0.001, 0.01, 0.1):
            x, h = run(I0, 2, alpha=a, I1=I1)
            print(shape, "SP a", a, " ".join(f"{v:.1e}" for v in h))
