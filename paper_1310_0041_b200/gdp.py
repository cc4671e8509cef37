"""Thin Python binding of the C ABI (include/gdp.h), same names, torch tensors in.

Marshalling only: tensors are passed as raw device (or host) pointers; every step of
the hot path runs in libgdp.so's kernels.  Volumes are torch tensors of shape
(nz, ny, nx), contiguous, slice-major (x fastest), uint8 or float32.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib as L


class GdpError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str):
        super().__init__(f"{where}: {L.STATUS.get(code, code)}: {msg}")
        self.code = code


def _check(code: int, where: str, allow_noconv: bool = False) -> int:
    if code == 0 or (allow_noconv and code == 3):
        return code
    raise GdpError(code, where, L.lib().gdp_last_error().decode())


def default_opts(**kw) -> L.Opts:
    o = L.Opts()
    _check(L.lib().gdp_opts_default(C.byref(o)), "gdp_opts_default")
    for k, v in kw.items():
        if not hasattr(o, k):
            raise AttributeError(f"gdp_opts has no field {k}")
        setattr(o, k, _scheme(v) if k == "scheme" else v)
    return o


def _dims(t: torch.Tensor) -> L.Dims:
    if t.dim() == 2:
        return L.Dims(t.shape[1], t.shape[0], 1)
    if t.dim() != 3:
        raise ValueError("volumes are (nz, ny, nx)")
    return L.Dims(t.shape[2], t.shape[1], t.shape[0])


def _dtype(t: torch.Tensor) -> int:
    if t.dtype == torch.uint8:
        return L.GDP_U8
    if t.dtype == torch.float32:
        return L.GDP_F32
    raise TypeError(f"unsupported dtype {t.dtype} (uint8 or float32)")


def _dev(t: torch.Tensor, name: str, dtypes=(torch.uint8, torch.float32)) -> int:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.dtype not in dtypes:
        raise TypeError(f"{name}: dtype {t.dtype} not in {dtypes}")
    return t.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def get_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (rank 0 creates it, every rank passes it to Ctx)."""
    buf = C.create_string_buffer(128)
    _check(L.lib().gdp_get_unique_id(buf, 128), "gdp_get_unique_id")
    return buf.raw


def partition(nz: int, world: int) -> list[tuple[int, int]]:
    """Even z-slab split in rank order [(z0, nz_local)], the split the loopback ctx uses."""
    base, rem = divmod(nz, world)
    out, z = [], 0
    for r in range(world):
        n = base + (1 if r < rem else 0)
        out.append((z, n))
        z += n
    return out


class Ctx:
    """gdp_ctx: per-device solver context (hierarchy cache, events, communicator)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_unique_id: bytes | None = None,
                 loopback: int = 0):
        self._p = C.c_void_p()
        lib = L.lib()
        if loopback:
            _check(lib.gdp_ctx_create_loopback(C.byref(self._p), device, loopback), "gdp_ctx_create_loopback")
        else:
            uid = None if nccl_unique_id is None else C.create_string_buffer(nccl_unique_id, len(nccl_unique_id))
            _check(lib.gdp_ctx_create(C.byref(self._p), device, rank, world, uid), "gdp_ctx_create")
        self.device, self.rank, self.world = device, rank, world

    @property
    def ptr(self):
        return self._p

    def close(self):
        if self._p:
            L.lib().gdp_ctx_destroy(self._p)
            self._p = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gdp_diffuse_z(ctx: Ctx, I0: torch.Tensor, I1: torch.Tensor | None = None, W=(1.0, 1.0, 0.1),
                  alpha: float = 0.0, z0_global: int = 0, nz_global: int | None = None, opts=None,
                  stream=None, check: bool = True):
    """Phase 1, Eq. (1).  Returns (I1, report dict)."""
    if I1 is None:
        I1 = torch.empty(I0.shape, dtype=torch.float32, device=I0.device)
    d = _dims(I0)
    rep = L.Report()
    o = opts if opts is not None else default_opts()
    rc = L.lib().gdp_diffuse_z(ctx.ptr, _dev(I0, "I0"), _dtype(I0), _dev(I1, "I1", (torch.float32,)), d,
                               z0_global, d.nz if nz_global is None else nz_global, L.Weights(*W), alpha,
                               C.byref(o), C.byref(rep), _stream(stream))
    if check:
        _check(rc, "gdp_diffuse_z", allow_noconv=True)
    return I1, rep.as_dict()


def gdp_screened_poisson_slices(ctx: Ctx, I0: torch.Tensor, I1: torch.Tensor, I2: torch.Tensor | None = None,
                                alpha: float = 0.01, opts=None, stream=None, check: bool = True):
    """Phase 2, Eq. (2), per slice.  Returns (I2, report dict)."""
    if I2 is None:
        I2 = torch.empty(I0.shape, dtype=torch.float32, device=I0.device)
    d = _dims(I0)
    rep = L.Report()
    o = opts if opts is not None else default_opts()
    rc = L.lib().gdp_screened_poisson_slices(ctx.ptr, _dev(I0, "I0"), _dtype(I0),
                                             _dev(I1, "I1", (torch.float32,)), _dev(I2, "I2", (torch.float32,)),
                                             d, alpha, C.byref(o), C.byref(rep), _stream(stream))
    if check:
        _check(rc, "gdp_screened_poisson_slices", allow_noconv=True)
    return I2, rep.as_dict()


def gdp_destripe(ctx: Ctx, I0: torch.Tensor, alpha: float = 0.01, W=(1.0, 1.0, 0.1), I1=None, I2=None,
                 z0_global: int = 0, nz_global: int | None = None, opts=None, stream=None):
    """Both phases.  Returns (I1, I2, report1, report2)."""
    if I1 is None:
        I1 = torch.empty(I0.shape, dtype=torch.float32, device=I0.device)
    if I2 is None:
        I2 = torch.empty(I0.shape, dtype=torch.float32, device=I0.device)
    d = _dims(I0)
    r1, r2 = L.Report(), L.Report()
    o = opts if opts is not None else default_opts()
    rc = L.lib().gdp_destripe(ctx.ptr, _dev(I0, "I0"), _dtype(I0), _dev(I1, "I1", (torch.float32,)),
                              _dev(I2, "I2", (torch.float32,)), d, z0_global,
                              d.nz if nz_global is None else nz_global, L.Weights(*W), alpha, C.byref(o),
                              C.byref(r1), C.byref(r2), _stream(stream))
    _check(rc, "gdp_destripe", allow_noconv=True)
    return I1, I2, r1.as_dict(), r2.as_dict()


def gdp_destripe_host(ctx: Ctx, I0: torch.Tensor, I2: torch.Tensor, I1: torch.Tensor | None = None,
                      alpha: float = 0.01, W=(1.0, 1.0, 0.1), hbm_budget_bytes: int = 0, opts=None,
                      z0_global: int = 0, nz_global: int | None = None):
    """Host-buffer entry (a13): CPU tensors in (pinned for async copies), CPU tensors out."""
    for t, nm in ((I0, "I0"), (I2, "I2")) + (((I1, "I1"),) if I1 is not None else ()):
        if t.is_cuda or not t.is_contiguous():
            raise ValueError(f"{nm} must be a contiguous host tensor")
    d = _dims(I0)
    r1, r2 = L.Report(), L.Report()
    o = opts if opts is not None else default_opts()
    rc = L.lib().gdp_destripe_host(ctx.ptr, I0.data_ptr(), _dtype(I0), None if I1 is None else I1.data_ptr(),
                                   I2.data_ptr(), d, z0_global, d.nz if nz_global is None else nz_global,
                                   L.Weights(*W), alpha, hbm_budget_bytes, C.byref(o), C.byref(r1), C.byref(r2))
    _check(rc, "gdp_destripe_host", allow_noconv=True)
    return r1.as_dict(), r2.as_dict()


def gdp_npr_filter(ctx: Ctx, I0: torch.Tensor, out: torch.Tensor | None = None, W=(1.0, 1.0, 0.1),
                   alpha: float = 0.001, lam: float = 1.25, sigma: float = 5.0 / 255.0, opts=None,
                   stream=None, check: bool = True):
    """NEXT-1: the §6 NPR filter.  Returns (out, report dict)."""
    if out is None:
        out = torch.empty(I0.shape, dtype=torch.float32, device=I0.device)
    d = _dims(I0)
    rep = L.Report()
    o = opts if opts is not None else default_opts()
    rc = L.lib().gdp_npr_filter(ctx.ptr, _dev(I0, "I0"), _dtype(I0), _dev(out, "out", (torch.float32,)), d,
                                L.Weights(*W), alpha, lam, sigma, C.byref(o), C.byref(rep), _stream(stream))
    if check:
        _check(rc, "gdp_npr_filter", allow_noconv=True)
    return out, rep.as_dict()


def gdp_vcycle(ctx: Ctx, x: torch.Tensor, b: torch.Tensor, W=(1.0, 1.0, 0.1), alpha: float = 0.0,
               z0_global: int = 0, nz_global: int | None = None, opts=None, stream=None) -> float:
    """One V-cycle on (alpha - div W grad) x = b.  Returns rel-res after."""
    d = _dims(x)
    rel = C.c_double()
    o = opts if opts is not None else default_opts()
    _check(L.lib().gdp_vcycle(ctx.ptr, _dev(x, "x", (torch.float32,)), _dev(b, "b", (torch.float32,)), d,
                              z0_global, d.nz if nz_global is None else nz_global, L.Weights(*W), alpha,
                              C.byref(o), C.byref(rel), _stream(stream)), "gdp_vcycle")
    return rel.value


def gdp_residual(ctx: Ctx, x: torch.Tensor, b: torch.Tensor, r: torch.Tensor | None = None, W=(1.0, 1.0, 0.1),
                 alpha: float = 0.0, z0_global: int = 0, nz_global: int | None = None, stream=None):
    """r = b - A x with fp64 norms.  Returns (r or None, ||r||^2, ||b||^2)."""
    d = _dims(x)
    nr, nb = C.c_double(), C.c_double()
    _check(L.lib().gdp_residual(ctx.ptr, _dev(x, "x", (torch.float32,)), _dev(b, "b", (torch.float32,)),
                                None if r is None else _dev(r, "r", (torch.float32,)), d, z0_global,
                                d.nz if nz_global is None else nz_global, L.Weights(*W), alpha,
                                C.byref(nr), C.byref(nb), _stream(stream)), "gdp_residual")
    return r, nr.value, nb.value


def _scheme(s) -> int:
    return L.SCHEMES[s] if isinstance(s, str) else int(s)


def gdp_scheme_levels(ctx: Ctx, scheme, dims, W=(1.0, 1.0, 0.1), alpha: float = 0.0, per_slice: bool = False,
                      opts=None) -> list[dict]:
    """NEXT-3 hierarchy of a Hybrid / Linear solve: [{dims (nz, ny, nx), coarsened (x, y, z)}] per level."""
    nz, ny, nx = dims
    n = C.c_int()
    ld = (L.Dims * 32)()
    co = (C.c_int * 96)()
    o = opts if opts is not None else default_opts()
    _check(L.lib().gdp_scheme_levels(ctx.ptr, _scheme(scheme), L.Dims(nx, ny, nz), L.Weights(*W), alpha,
                                     int(per_slice), C.byref(o), C.byref(n), ld, co, 32), "gdp_scheme_levels")
    return [{"dims": (ld[i].nz, ld[i].ny, ld[i].nx), "coarsened": tuple(bool(co[3 * i + d]) for d in range(3))}
            for i in range(n.value)]


def gdp_scheme_apply(ctx: Ctx, scheme, level: int, x: torch.Tensor, y: torch.Tensor | None = None,
                     fine_dims=None, W=(1.0, 1.0, 0.1), alpha: float = 0.0, per_slice: bool = False, opts=None,
                     stream=None) -> torch.Tensor:
    """y = A_level x of a Hybrid / Linear hierarchy built for `fine_dims` (nz, ny, nx)."""
    nz, ny, nx = fine_dims
    y = torch.empty_like(x) if y is None else y
    o = opts if opts is not None else default_opts()
    _check(L.lib().gdp_scheme_apply(ctx.ptr, _scheme(scheme), level, _dev(x, "x", (torch.float32,)),
                                    _dev(y, "y", (torch.float32,)), L.Dims(nx, ny, nz), L.Weights(*W), alpha,
                                    int(per_slice), C.byref(o), _stream(stream)), "gdp_scheme_apply")
    return y


def gdp_scheme_residual(ctx: Ctx, scheme, x: torch.Tensor, b: torch.Tensor, r: torch.Tensor | None = None,
                        W=(1.0, 1.0, 0.1), alpha: float = 0.0, per_slice: bool = False, stream=None):
    """r = b - A x of the scheme's finest operator; returns (r or None, ||r||^2, ||b||^2)."""
    d = _dims(x)
    nr, nb = C.c_double(), C.c_double()
    _check(L.lib().gdp_scheme_residual(ctx.ptr, _scheme(scheme), _dev(x, "x", (torch.float32,)),
                                       _dev(b, "b", (torch.float32,)),
                                       None if r is None else _dev(r, "r", (torch.float32,)), d, L.Weights(*W),
                                       alpha, int(per_slice), C.byref(nr), C.byref(nb), _stream(stream)),
           "gdp_scheme_residual")
    return r, nr.value, nb.value


def profile_begin() -> None:
    """Start per-kernel-class device timing (gdp_profile_begin)."""
    _check(L.lib().gdp_profile_begin(), "gdp_profile_begin")


def profile_end() -> list[dict]:
    """Stop timing; returns [{name, launches, ms, alg_bytes}] per kernel class."""
    arr = (L.KernelStat * 48)()
    n = C.c_int()
    _check(L.lib().gdp_profile_end(arr, 48, C.byref(n)), "gdp_profile_end")
    return [{"name": arr[i].name.decode(), "launches": arr[i].launches, "ms": arr[i].ms,
             "alg_bytes": arr[i].alg_bytes, "alg_bytes_8d": arr[i].alg_bytes_8d} for i in range(n.value)]


def kernel_launch_count() -> int:
    return int(L.lib().gdp_kernel_launch_count())


def version() -> str:
    return L.lib().gdp_version().decode()
