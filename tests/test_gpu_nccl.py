"""The NCCL data plane of pipeline.DeviceSimulation executed on the B200:
torchrun, backend "nccl", E/B broadcast + exact int64 moment all-reduce and
reduce-to-root, compared bitwise with the non-distributed run
(tests/dist_nccl_check.py).  One GPU is available to this build, so the
world size is 1 (N>1 host logic: tests/test_multiproc.py, gloo)."""

import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
def test_nccl_world1_broadcast_and_reduce(gpu):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "dist_nccl_check.py")]
    env = dict(os.environ, NCCL_DEBUG="WARN")
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    assert "NCCL_OK backend=nccl world=1 cases=4" in r.stdout, (r.stdout + r.stderr)[-4000:]
