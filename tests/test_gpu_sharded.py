"""The SFC-sharded multi-GPU driver, run as 2 or 4 ranks sharing one B200 over
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


@pytest.mark.parametrize("name,overlap,l1tile,ranks", [("C2", "0", "32", 2), ("C2", "1", "0", 2), ("C3", "0", "16", 2),
                                                       ("C4", "1", "16", 2), ("C5", "0", "32", 2),
                                                       ("C4", "1", "16", 4), ("C5", "1", "16", 4)])
def test_sharded_ranks_match_single_gpu(name, overlap, l1tile, ranks):
    """overlap = MLAMR_OVERLAP_REFRESH: the parents' refresh (ii) on its own
    stream, overlapping the step.  l1tile = MLAMR_L1_TILE: level 1 cut into
    tiles of that many cells a side and spread over the ranks ("0": the
    single level-1 patch, owned by rank 0); the single-GPU run the worker
    compares with uses the same level-1 layout, and
    test_gpu_driver.py::test_tiled_level1_is_bit_identical ties that to the
    untiled run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ranks}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(HERE, "dist_gpu_worker.py"), name]
    env = dict(os.environ, MLAMR_OVERLAP_REFRESH=overlap, MLAMR_L1_TILE=l1tile)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=420, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("sharded == single-GPU") == ranks, r.stdout[-2000:]
