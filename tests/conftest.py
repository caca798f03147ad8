import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "golden_moekit.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running test")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


def bf16_round(a):
    """float32 -> bfloat16 (RNE) values, returned as float32."""
    f = np.ascontiguousarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


@pytest.fixture(scope="session")
def cuda():
    """Skip-free GPU gate: on a GPU box the library MUST load; a missing
    library is a failure, not a skip."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2508_07329_b200 import _lib
    _lib.load()
    return torch.device("cuda:0")


@pytest.fixture(params=["warp", "cta"])
def k1_kernel(request, cuda):
    """Run a K1 test through each of the bit-identical per-token kernels:
    the per-warp / bulk kernels ("warp") and the CTA-per-row kernel the
    library picks for small row counts ("cta")."""
    from paper_2508_07329_b200 import _lib
    with _lib.tuned(_lib.TUNE_K1_SMALL_ROWS, 0 if request.param == "warp" else 1 << 40):
        yield request.param
