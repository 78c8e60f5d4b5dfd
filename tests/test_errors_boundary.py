"""The drop-in error contract: with the reference package
importable, the shims raise the reference's own exception classes
(src/errors.py:4-37), so the reference's handlers -- run_simulation's
abort dump (src/driver.py:394-401) and the CLI's exit codes
(src/cli.py:126-134) -- catch a GPU-side CFL violation or non-finite
abort.  Run in a subprocess so the reference never enters this process
(nothing on the GPU box may read /root/reference)."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

REF_SRC = "/root/reference/pkg/src"

_PROBE = r"""
import sys
sys.path.insert(0, {root!r})
sys.path.insert(0, {ref!r})
import mlamr.errors as R
from paper_1803_01450_b200 import errors as E, config, frames
assert E.FROM_REFERENCE
for n in ("MlamrError", "ConfigError", "NotRefinedError", "GeometryError", "TimeSyncError",
          "CflViolationError", "NumericalAbortError", "FrameFormatError"):
    assert getattr(E, n) is getattr(R, n), n
assert config.ConfigError is R.ConfigError and frames.FrameFormatError is R.FrameFormatError
# the device status word maps onto the reference's classes: the reference's
# own `except CflViolationError` / `except NumericalAbortError` catch them
from paper_1803_01450_b200._native import ST_CFL, ST_GEOMETRY, ST_NONFINITE
for bit, cls in ((ST_CFL, R.CflViolationError), (ST_GEOMETRY, R.GeometryError),
                 (ST_NONFINITE, R.NumericalAbortError)):
    try:
        E.raise_status(bit, "probe")
    except (R.NumericalAbortError, R.CflViolationError, R.GeometryError) as exc:
        assert type(exc) is cls, (bit, type(exc))
    else:
        raise AssertionError(bit)
print("ok")
"""


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present (GPU box)")
def test_shims_raise_the_reference_exception_classes():
    env = dict(os.environ, NUMBA_CACHE_DIR="/tmp/numba_cache")
    out = subprocess.run([sys.executable, "-c", _PROBE.format(root=ROOT, ref=REF_SRC)],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-3000:]
    assert out.stdout.strip().endswith("ok")


def test_local_exception_classes_mirror_the_reference():
    """Without the reference on the path: same names, hierarchy and the
    ConfigError(key, message) constructor."""
    from paper_1803_01450_b200 import errors as E
    for n in ("ConfigError", "NotRefinedError", "GeometryError", "TimeSyncError",
              "CflViolationError", "NumericalAbortError", "FrameFormatError"):
        assert issubclass(getattr(E, n), E.MlamrError), n
    e = E.ConfigError("domain.nx", "must be positive")
    assert e.key == "domain.nx" and str(e) == "domain.nx: must be positive"


def test_oracle_rejects_non_telescoping_bathymetry(oracle):
    """The oracle's check_bathymetry_consistency (coarsen.py:79-100) under
    C2's fixed level-2 tiling: a 1e-9 m perturbation under a level-2 patch
    raises AssertionError, one outside every patch is never checked."""
    import numpy as np
    import pytest
    from paper_1803_01450_b200 import problems

    def perturbed(j, i):
        pb = problems.config2(n_coarse_steps=1)
        fine = np.array(pb.bathy_levels[1], copy=True)
        fine[j, i] += 1e-9
        pb.bathy_levels = [pb.bathy_levels[0], fine]
        return pb

    with pytest.raises(AssertionError):
        oracle.Simulation(perturbed(200, 300))
    oracle.Simulation(perturbed(10, 20))
