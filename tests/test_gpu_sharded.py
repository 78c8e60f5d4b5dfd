"""The SFC-sharded multi-GPU driver, run as 2 ranks sharing one B200 over
the gloo backend (host-staged exchanges; kernels never wait on another
rank), must reproduce the single-GPU run bit for bit."""

import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name,overlap", [("C2", "0"), ("C2", "1"), ("C3", "0"), ("C4", "1"), ("C5", "0")])
def test_sharded_two_ranks_match_single_gpu(name, overlap):
    """overlap = MLAMR_OVERLAP_REFRESH: the parents' refresh (ii) on its own
    stream, overlapping the step."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(HERE, "dist_gpu_worker.py"), name]
    env = dict(os.environ, MLAMR_OVERLAP_REFRESH=overlap)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=420, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("sharded == single-GPU") == 2, r.stdout[-2000:]
