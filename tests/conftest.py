import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# every 3D level takes the fused z-march in the schedule tests (the library default hands levels under
# 2M cells to the reference kernels, which would make small fused-vs-reference comparisons vacuous)
os.environ.setdefault("GDP_F3D_MIN", "0")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def gpu_ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device")
    import paper_1310_0041_b200 as gdp
    ctx = gdp.Ctx(0)
    yield ctx
    ctx.close()
