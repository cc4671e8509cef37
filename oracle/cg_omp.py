"""ctypes binding of oracle/cg_omp.c (C + OpenMP fp64 CG oracle) — TEST INFRASTRUCTURE ONLY.

Same definitions as oracle/gdp_oracle.py (operators assembled link by link, Neumann, CG to 1e-10,
phase-1 mean pin), written in C so that bench.py can time the oracle on ALL host cores as the
CPU baseline (SURVEY.md §8(d) "Oracle timing beside the GPU").  Pinned against gdp_oracle in
tests/test_oracle_cg_omp.py.  Only tests/, __graft_entry__ and bench.py's CPU legs use it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cg_omp.c")
LIB = os.path.join(HERE, "libgdp_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """gcc -O3 -fopenmp (portable code generation: the GPU box's host CPU may differ)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + ".tmp"
        subprocess.run(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-o", tmp, SRC, "-lm"], check=True)
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d = C.POINTER(C.c_double)
        i64 = C.c_longlong
        _lib.gdp_oracle_diffuse_z.argtypes = [d, d, i64, i64, i64, C.c_double, C.c_double, C.c_double, C.c_double,
                                              C.c_int]
        _lib.gdp_oracle_slices.argtypes = [d, d, d, i64, i64, i64, C.c_double, C.c_double, C.c_int]
        _lib.gdp_oracle_threads.restype = C.c_int
    return _lib


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(I0):
    I0 = np.asarray(I0)
    if I0.dtype == np.uint8:  # reading c-9: u8/255 rounded to fp32
        return np.ascontiguousarray((I0.astype(np.float32) / np.float32(255.0)).astype(np.float64))
    return np.ascontiguousarray(I0, dtype=np.float64) if I0.dtype == np.float64 else \
        np.ascontiguousarray(I0.astype(np.float32).astype(np.float64))


def threads() -> int:
    return int(lib().gdp_oracle_threads())


def diffuse_z(I0, W=(1.0, 1.0, 0.1), tol=1e-10, maxit=200000, return_iters=False):
    """Phase 1 (Eq. 1), the definition of oracle.gdp_oracle.diffuse_z on all OpenMP threads."""
    I = _f64(I0)
    nz, ny, nx = I.shape
    out = np.empty_like(I)
    it = lib().gdp_oracle_diffuse_z(_p(I), _p(out), nx, ny, nz, W[0], W[1], W[2], tol, maxit)
    if it < 0:
        raise RuntimeError(f"gdp_oracle_diffuse_z failed ({it})")
    return (out, it) if return_iters else out


def screened_poisson_slices(I0, I1, alpha=0.01, tol=1e-10, maxit=200000, return_iters=False):
    """Phase 2 (Eq. 2) per slice, the definition of oracle.gdp_oracle.screened_poisson_slices."""
    I = _f64(I0)
    J = np.ascontiguousarray(I1, dtype=np.float64)
    nz, ny, nx = I.shape
    out = np.empty_like(I)
    it = lib().gdp_oracle_slices(_p(I), _p(J), _p(out), nx, ny, nz, alpha, tol, maxit)
    if it < 0:
        raise RuntimeError(f"gdp_oracle_slices failed ({it})")
    return (out, it) if return_iters else out


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
