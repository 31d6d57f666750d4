"""pytest plugin (``-p bp_install``) for running the REFERENCE's own test
files with the B200 kernels bound into ``batchpic.kernels``.

Loaded before test collection, so every reference module that resolves
``kernels.fused_span`` / ``push_span`` / ``deposit_span`` / ``gather_span``
at call time (mover.py:85,135,154,179,194,221; pipeline.py:206;
test_acceptance.py:84-109) reaches ``paper_2008_04397_b200.kernels``.
It fails loudly without a GPU: there is no CPU fallback to hide behind.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import torch  # noqa: E402

assert torch.cuda.is_available(), "bp_install: the drop-in suite needs a CUDA device"

import batchpic.kernels as _ref_kernels  # noqa: E402
from paper_2008_04397_b200 import kernels as _bp  # noqa: E402

_bp.install(_ref_kernels)
CALLS = {"fused_span": 0, "push_span": 0, "deposit_span": 0, "gather_span": 0}


def _counting(name):
    fn = getattr(_ref_kernels, name)

    def wrapped(*a, **k):
        CALLS[name] += 1
        return fn(*a, **k)

    wrapped.__name__ = name
    return wrapped


for _n in CALLS:
    setattr(_ref_kernels, _n, _counting(_n))


def pytest_terminal_summary(terminalreporter):
    assert _ref_kernels.fused_span.__name__ == "fused_span"
    terminalreporter.write_line(
        "bp_install: B200 kernel calls " + " ".join(f"{k}={v}" for k, v in CALLS.items()))
