"""Seeded synthetic EM-like voxel stacks — the ONE module both sides share.

This module holds no arithmetic of the paper's method (no stencil, no gradient
field, no solver).  It only produces the input bytes that the CPU oracle
(`oracle/`) and the CUDA path (`paper_1310_0041_b200/`) both consume, so that
parity is checked on identical inputs.

Recipe (BASELINE.json configs):
  per slice z, an RNG keyed by (seed, z) — numpy PCG64 via default_rng([seed, z]);
  draws, in this order:
    w      ~ N(0,1) per pixel (ny, nx)        -> texture t = gauss(w, sigma=4, reflect),
                                                 rescaled to mean 0.5, std 0.15
    lines  20 x (x0, y0, x1, y1) ~ U[0,nx)/U[0,ny) -> 1-px segments, t -= 0.4 on them
    g      ~ U(0.8, 1.2)   slice gain
    o      ~ N(0, 0.05)    slice offset
    theta  ~ U(0, 2 pi)    illumination-ramp direction, ramp = 0.1(cos th xh + sin th yh)
    noise  ~ N(0, 0.02) per pixel
  s = clip(t*g + o + ramp + noise, 0, 1)
  fp32 configs keep s as float32; u8 configs store rint(255 s) (round-half-even).

The paper's data (Mouse S1) is not available; these stacks
stand in for it with the shapes BASELINE.json names.
"""
from __future__ import annotations

import numpy as np

try:  # scipy is only needed for the texture blur
    from scipy.ndimage import gaussian_filter as _gauss
except Exception:  # pragma: no cover
    _gauss = None

N_LINES = 20

# BASELINE.json "configs" (index = config number)
CONFIGS = {
    0: dict(name="c0_tiny_64x64x16_f32", nx=64, ny=64, nz=16, dtype="f32", alphas=(0.01,), seed=0),
    1: dict(name="c1_1024x1024x128_u8", nx=1024, ny=1024, nz=128, dtype="u8",
            alphas=(0.001, 0.01, 0.1), seed=1),
    2: dict(name="c2_slice_21496x25792_f32", nx=21496, ny=25792, nz=1, dtype="f32",
            alphas=(0.01,), seed=2),
    3: dict(name="c3_4096x4096x512_u8", nx=4096, ny=4096, nz=512, dtype="u8", alphas=(0.01,), seed=3),
    4: dict(name="c4_16384x16384x1024_u8", nx=16384, ny=16384, nz=1024, dtype="u8",
            alphas=(0.01,), seed=4),
}


def _line_pixels(x0, y0, x1, y1, nx, ny):
    n = int(np.ceil(max(abs(x1 - x0), abs(y1 - y0)))) + 1
    t = np.linspace(0.0, 1.0, n)
    xs = np.clip(np.rint(x0 + t * (x1 - x0)).astype(np.int64), 0, nx - 1)
    ys = np.clip(np.rint(y0 + t * (y1 - y0)).astype(np.int64), 0, ny - 1)
    return ys, xs


def make_slice(nx: int, ny: int, seed: int, z: int) -> np.ndarray:
    """One float64 slice s in [0,1], shape (ny, nx)."""
    rng = np.random.default_rng([int(seed), int(z)])
    w = rng.standard_normal((ny, nx))
    if _gauss is None:
        raise RuntimeError("scipy is required for the synthetic texture")
    t = _gauss(w, sigma=4.0, mode="reflect")
    sd = t.std()
    t = 0.5 + 0.15 * (t - t.mean()) / (sd if sd > 0 else 1.0)
    pts = rng.random((N_LINES, 4))
    for k in range(N_LINES):
        ys, xs = _line_pixels(pts[k, 0] * nx, pts[k, 1] * ny, pts[k, 2] * nx, pts[k, 3] * ny, nx, ny)
        t[ys, xs] -= 0.4
    g = rng.uniform(0.8, 1.2)
    o = rng.normal(0.0, 0.05)
    th = rng.uniform(0.0, 2.0 * np.pi)
    xh = (np.arange(nx) / max(nx - 1, 1) - 0.5)[None, :]
    yh = (np.arange(ny) / max(ny - 1, 1) - 0.5)[:, None]
    ramp = 0.1 * (np.cos(th) * xh + np.sin(th) * yh)
    noise = rng.normal(0.0, 0.02, (ny, nx))
    return np.clip(t * g + o + ramp + noise, 0.0, 1.0)


def make_stack(nx: int, ny: int, nz: int, seed: int, dtype: str = "f32") -> np.ndarray:
    """Slice-major stack, shape (nz, ny, nx) (x fastest), dtype float32 or uint8."""
    if dtype not in ("f32", "u8"):
        raise ValueError(dtype)
    out = np.empty((nz, ny, nx), dtype=np.float32 if dtype == "f32" else np.uint8)
    for z in range(nz):
        s = make_slice(nx, ny, seed, z)
        if dtype == "f32":
            out[z] = s.astype(np.float32)
        else:
            out[z] = np.rint(255.0 * s).astype(np.uint8)
    return out


def make_config(k: int, nz: int | None = None, crop: tuple[int, int] | None = None) -> np.ndarray:
    """Input stack of BASELINE.json config k (optionally fewer slices / xy crop for samples)."""
    c = CONFIGS[k]
    nx, ny = (c["nx"], c["ny"]) if crop is None else crop
    return make_stack(nx, ny, c["nz"] if nz is None else nz, c["seed"], c["dtype"])


def offset_striped_u8(nx: int, ny: int, nz: int, seed: int) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Closed-form input I0 = T(x,y) + c(z) built in u8 units.

    T_u8 in [20,235] from one generated slice, c_u8(z) integers in [-20,20]; no clipping
    occurs, so I0 = (T_u8 + c_u8)/255 is exactly separable.  Returns (I0_u8, T_u8, c_u8).
    """
    s = make_slice(nx, ny, seed, 0)
    T = (20 + np.rint(215.0 * s)).astype(np.int32)
    rng = np.random.default_rng([int(seed), 1 << 20])
    c = rng.integers(-20, 21, size=nz).astype(np.int32)
    I0 = (T[None, :, :] + c[:, None, None]).astype(np.uint8)
    return I0, T, c


def random_field(shape, seed: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    """Plain U(lo,hi) float32 field (for unit-level parity cases)."""
    rng = np.random.default_rng([int(seed), 7777])
    return (lo + (hi - lo) * rng.random(shape)).astype(np.float32)



def cosine_mode(i: np.ndarray, k: int, n: int) -> np.ndarray:
    """Neumann cosine mode cos(pi k (i + 1/2) / n) at integer cells i (fp64)."""
    return np.cos(np.pi * k * (np.asarray(i, dtype=np.float64) + 0.5) / n)


def cosine_modes(shape, modes, amps, c0: float = 0.5, block: int = 512) -> np.ndarray:
    """fp32 stack c0 + sum_j amps[j] * phi_kj(x) phi_lj(y) phi_mj(z), shape (nz, ny, nx), built in
    row blocks (config-2 slices do not fit fp64 temporaries).  modes: list of (k, l, m)."""
    nz, ny, nx = shape
    out = np.empty(shape, dtype=np.float32)
    fx = [cosine_mode(np.arange(nx), k, nx) for k, _, _ in modes]
    fz = [cosine_mode(np.arange(nz), m, nz) for _, _, m in modes]
    for z in range(nz):
        for y0 in range(0, ny, block):
            ys = np.arange(y0, min(y0 + block, ny))
            acc = np.full((len(ys), nx), c0, dtype=np.float64)
            for j, (k, l, m) in enumerate(modes):
                acc += (amps[j] * fz[j][z]) * np.outer(cosine_mode(ys, l, ny), fx[j])
            out[z, y0:y0 + len(ys)] = acc.astype(np.float32)
    return out
