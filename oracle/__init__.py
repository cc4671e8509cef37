"""CPU ORACLE for arxiv 1310.0041 — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import anything under `oracle/`.  The product
package `paper_1310_0041_b200` never imports it and has no CPU fallback.

The oracle shares no code with the CUDA path: it assembles the paper's discrete
operators from forward differences on links (gradient) and their negative
transposes (divergence) and solves them with plain conjugate gradient in fp64
(`gdp_oracle`), with an independent closed-form DCT-II eigen-solver
(`closed_form`) and a brute-force energy-Hessian assembly for tiny grids
(`brute`) as pins.  See DESIGN.md "Oracle" for every reading of the paper.
"""
from .gdp_oracle import (  # noqa: F401
    decode,
    forward_difference,
    gradient,
    divergence,
    apply_A,
    rhs_general,
    rhs_diffusion,
    rhs_blend,
    cg,
    diffuse_z,
    screened_poisson_slices,
    destripe,
    residual,
    rel_residual,
    npr_gradient_field,
    rhs_npr,
    npr_filter,
    slice_rel_residuals,
)
from .closed_form import (  # noqa: F401
    path_eigenvalues,
    dct_solve,
    diffuse_z_dct,
    screened_poisson_slices_dct,
    ad_gain,
    sp_gain,
    combined_gain,
)
