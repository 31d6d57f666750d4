"""The reference's OWN tests, run with the B200 kernels installed into
``batchpic.kernels`` (``kernels.install()``): the drop-in proven inside the
reference's callers — its mover wrappers (pkg/src/batchpic/mover.py), its
cycle driver (pipeline.py:206) and its acceptance scenarios.

Needs ``baseline/_ref`` (scripts/stage_reference.sh: a pip install of
/root/reference/pkg plus a copy of pkg/tests; git-ignored, travels to the
GPU box).  Each file runs in a subprocess with the plugin
tests/refsuite/bp_install.py loaded before collection.
"""

import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "ref_tests")

# (file, -k expression or None): the hot-path and pipeline suites in full,
# and the acceptance scenarios that go through the kernel seam
SUITES = [
    ("test_mover.py", None),          # weights, gather, corrector, mover, deposit, fusion
    ("test_pipeline.py", None),       # sequential-reference bitwise, G/M invariance, sorting
    # C1..C11 acceptance scenarios.  C12's speedup floor times the reference's
    # CPU worker pool (4 workers >= 1.3x 1 worker, test_acceptance.py:548-555);
    # with the kernels installed all workers share one GPU, so that floor
    # measures host thread contention, not the kernel seam
    ("test_acceptance.py", "not test_c12_benchmark_harness"),
    ("test_diagnostics.py", None),    # mixed-mode gather (test_diagnostics.py:32-67)
    ("test_particles.py", None),
    ("test_fields.py", None),
]


def _run(fname, kexpr):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join(
        [os.path.join(ROOT, "tests", "refsuite"), REF, ROOT, env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "bp_install", "-p", "no:cacheprovider",
           "--rootdir", REF_TESTS, os.path.join(REF_TESTS, fname)]
    if kexpr:
        cmd += ["-k", kexpr]
    return subprocess.run(cmd, cwd=REF_TESTS, env=env, capture_output=True, text=True,
                          timeout=1800)


@pytest.mark.gpu
@pytest.mark.parametrize("fname,kexpr", SUITES, ids=[s[0] for s in SUITES])
def test_reference_suite_on_b200(gpu, fname, kexpr):
    assert os.path.isdir(REF_TESTS), (
        "baseline/_ref/ref_tests missing: run scripts/stage_reference.sh before pushing")
    r = _run(fname, kexpr)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    m = re.search(r"bp_install: B200 kernel calls (.*)", r.stdout)
    assert m, tail
    calls = dict(kv.split("=") for kv in m.group(1).split())
    print(fname, m.group(1), re.findall(r"\d+ passed.*", r.stdout)[-1:])
    if fname in ("test_mover.py", "test_pipeline.py", "test_acceptance.py"):
        assert int(calls["fused_span"]) > 0, "the suite never reached the B200 fused kernel"
