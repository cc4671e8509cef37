"""B200-native multigrid hot path of arXiv 1310.0041 (gradient-domain EM-stack processing).

The product is the C-ABI library `libgdp.so` (include/gdp.h) with hand-written sm_100a
kernels; this package is its thin Python binding.  It never imports `oracle/` and has
no CPU fallback.
"""
from .gdp import (  # noqa: F401
    Ctx,
    GdpError,
    default_opts,
    gdp_destripe,
    gdp_destripe_host,
    gdp_diffuse_z,
    gdp_npr_filter,
    gdp_residual,
    gdp_scheme_apply,
    gdp_scheme_levels,
    gdp_scheme_residual,
    gdp_screened_poisson_slices,
    gdp_vcycle,
    get_unique_id,
    partition,
    kernel_launch_count,
    profile_begin,
    profile_end,
    version,
)
