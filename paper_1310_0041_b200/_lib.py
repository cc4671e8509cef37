"""ctypes view of libgdp.so — the C ABI declared in include/gdp.h (argument marshalling only).

There is no fallback: if the in-tree library is missing or fails to load, every call
raises.  Build it with `python -m paper_1310_0041_b200.build`.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgdp.so")

GDP_MAX_CYCLES = 64

STATUS = {0: "GDP_OK", 1: "GDP_EINVAL", 2: "GDP_ECUDA", 3: "GDP_ENOCONV", 4: "GDP_ENOMEM", 5: "GDP_ENCCL"}
GDP_U8, GDP_F32 = 0, 1

# every symbol include/gdp.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "gdp_opts_default", "gdp_ctx_create", "gdp_ctx_create_loopback", "gdp_ctx_destroy",
    "gdp_diffuse_z", "gdp_screened_poisson_slices", "gdp_destripe", "gdp_destripe_host",
    "gdp_vcycle", "gdp_residual", "gdp_last_error", "gdp_version", "gdp_kernel_launch_count",
    "gdp_profile_begin", "gdp_profile_end", "gdp_get_unique_id", "gdp_npr_filter",
    "gdp_scheme_levels", "gdp_scheme_apply", "gdp_scheme_residual",
]
GDP_SCHEME_CONSTANT, GDP_SCHEME_HYBRID, GDP_SCHEME_LINEAR = 0, 1, 2
SCHEMES = {"constant": 0, "hybrid": 1, "linear": 2}


class Dims(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64)]


class Weights(C.Structure):
    _fields_ = [("bx", C.c_float), ("by", C.c_float), ("bz", C.c_float)]


class Opts(C.Structure):
    _fields_ = [("rel_tol", C.c_double), ("max_vcycles", C.c_int), ("nu_pre", C.c_int),
                ("nu_post", C.c_int), ("coarse_max", C.c_int), ("stagnation", C.c_int),
                ("fused", C.c_int), ("use_graphs", C.c_int), ("nu_pre_slices", C.c_int),
                ("nu_post_slices", C.c_int), ("omega", C.c_float), ("omega_slices", C.c_float),
                ("fmg", C.c_int), ("fmg_slices", C.c_int), ("dx_tol", C.c_double), ("scheme", C.c_int),
                ("half_staging", C.c_int), ("stream_fuse", C.c_int)]


class Report(C.Structure):
    _fields_ = [("status", C.c_int), ("vcycles", C.c_int), ("levels", C.c_int),
                ("rel_res", C.c_double * (GDP_MAX_CYCLES + 1)), ("norm_b", C.c_double),
                ("seconds", C.c_double), ("hbm_bytes_est", C.c_double),
                ("kernel_launches", C.c_int64), ("dx_inf", C.c_double)]

    def as_dict(self) -> dict:
        k = self.vcycles
        return {"status": STATUS.get(self.status, self.status), "vcycles": k, "levels": self.levels,
                "rel_res": [self.rel_res[i] for i in range(k + 1)], "norm_b": self.norm_b,
                "seconds": self.seconds, "hbm_bytes_est": self.hbm_bytes_est,
                "kernel_launches": self.kernel_launches, "dx_inf": self.dx_inf}


class KernelStat(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("ms", C.c_double),
                ("alg_bytes", C.c_double), ("alg_bytes_8d", C.c_double)]


_lib = None


def lib():
    """Load libgdp.so (raises if it is absent: the product path has no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1310_0041_b200.build`")
    L = C.CDLL(LIB_PATH)
    vp, i64, f32, i32 = C.c_void_p, C.c_int64, C.c_float, C.c_int
    P = C.POINTER
    sig = {
        "gdp_opts_default": ([P(Opts)], i32),
        "gdp_ctx_create": ([P(vp), i32, i32, i32, vp], i32),
        "gdp_ctx_create_loopback": ([P(vp), i32, i32], i32),
        "gdp_ctx_destroy": ([vp], i32),
        "gdp_diffuse_z": ([vp, vp, i32, vp, Dims, i64, i64, Weights, f32, P(Opts), P(Report), vp], i32),
        "gdp_screened_poisson_slices": ([vp, vp, i32, vp, vp, Dims, f32, P(Opts), P(Report), vp], i32),
        "gdp_destripe": ([vp, vp, i32, vp, vp, Dims, i64, i64, Weights, f32, P(Opts), P(Report),
                          P(Report), vp], i32),
        "gdp_destripe_host": ([vp, vp, i32, vp, vp, Dims, i64, i64, Weights, f32, C.c_size_t, P(Opts),
                               P(Report), P(Report)], i32),
        "gdp_vcycle": ([vp, vp, vp, Dims, i64, i64, Weights, f32, P(Opts), P(C.c_double), vp], i32),
        "gdp_npr_filter": ([vp, vp, i32, vp, Dims, Weights, f32, f32, f32, P(Opts), P(Report), vp], i32),
        "gdp_residual": ([vp, vp, vp, vp, Dims, i64, i64, Weights, f32, P(C.c_double), P(C.c_double), vp],
                         i32),
        "gdp_last_error": ([], C.c_char_p),
        "gdp_version": ([], C.c_char_p),
        "gdp_kernel_launch_count": ([], i64),
        "gdp_profile_begin": ([], i32),
        "gdp_get_unique_id": ([vp, C.c_size_t], i32),
        "gdp_profile_end": ([P(KernelStat), i32, P(i32)], i32),
        "gdp_scheme_levels": ([vp, i32, Dims, Weights, f32, i32, P(Opts), P(i32), P(Dims), P(i32), i32], i32),
        "gdp_scheme_apply": ([vp, i32, i32, vp, vp, Dims, Weights, f32, i32, P(Opts), vp], i32),
        "gdp_scheme_residual": ([vp, i32, vp, vp, vp, Dims, Weights, f32, i32, P(C.c_double), P(C.c_double), vp],
                                i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L
