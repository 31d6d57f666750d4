import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
MODES = {"double": (np.float64, np.float64), "single": (np.float32, np.float32),
         "mixed": (np.float32, np.float64)}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden(name):
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O


@pytest.fixture(scope="session")
def gpu():
    """The CUDA library and torch; fails loudly (never skips to a CPU path)
    when a test marked gpu runs without a device."""
    import torch
    assert torch.cuda.is_available(), "gpu test on a host without CUDA"
    from paper_2008_04397_b200 import _lib
    _lib.load()
    return torch
