"""C-ABI library: loads, exports every symbol include/gdp.h declares, host-side logic
that needs no GPU (defaults, argument validation, loud failure without a device)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "gdp.h")).read()
    return sorted(set(re.findall(r"^(?:int|int64_t|const char\*)\s+(gdp_\w+)\s*\(", src, re.M)))


def test_header_and_binding_agree():
    from paper_1310_0041_b200 import _lib
    assert _declared() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    from paper_1310_0041_b200 import _lib
    L = _lib.lib()
    for name in _declared():
        assert hasattr(L, name), name


def test_library_is_sm100a():
    import subprocess
    from paper_1310_0041_b200 import _lib
    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_opts_defaults():
    import paper_1310_0041_b200 as gdp
    o = gdp.default_opts()
    assert o.rel_tol == 1e-6 and o.max_vcycles == 30 and o.nu_pre == 2 and o.nu_post == 2
    assert o.coarse_max == 4096 and o.fused == 35
    assert o.nu_pre_slices == 1 and o.nu_post_slices == 2 and o.omega == 1.0
    assert o.fmg == 1 and o.fmg_slices == 3


def test_ctx_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("host-only check")
    import paper_1310_0041_b200 as gdp
    with pytest.raises(gdp.GdpError):
        gdp.Ctx(0)


def test_no_oracle_import_in_product():
    pkg = os.path.join(ROOT, "paper_1310_0041_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                s = open(os.path.join(dp, f)).read()
                assert "import oracle" not in s and "from oracle" not in s, f
