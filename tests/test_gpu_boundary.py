"""GPU side of the drop-in boundary: the threading
contract of the per-patch shims and the bathymetry telescoping check
(row A13, coarsen.py:79-100) on the device path."""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from conftest import load_golden, same
from gpu_util import HostPatch

pytestmark = pytest.mark.gpu


class _Params:
    def __init__(self, M, densities, g=1.0, tol=1e-3):
        self.num_layers = M
        self.densities = densities
        self.gravity = g
        self.dry_tolerance = tol


def _cases():
    z = load_golden("step_cases.npz")
    out = []
    for k in range(int(z["ncases"])):
        c = lambda key: z[f"c{k}_{key}"]
        M, nx, ny = int(c("M")), int(c("nx")), int(c("ny"))
        for s in range(4):
            out.append(dict(M=M, box=(0, 0, nx - 1, ny - 1), dx=float(c("dx")), dy=float(c("dy")),
                            h=c(f"s{s}_pre_h"), hu=c(f"s{s}_pre_hu"), hv=c(f"s{s}_pre_hv"), B=c("B"),
                            dt=float(c(f"s{s}_dt")), y_first=bool(c(f"s{s}_yfirst"))))
    return out


def test_step_patch_from_a_thread_pool_matches_serial_calls():
    """The reference maps step_patch over a level's patches with a
    ThreadPoolExecutor (driver.py:110, 231-232; numba nogil=True).  The
    shim called from 8 host threads at once on distinct patches gives the
    bits and results of serial calls."""
    from paper_1803_01450_b200 import ops
    cases = _cases()

    def mk(c):
        return HostPatch(c["box"], c["dx"], c["dy"], c["h"], c["hu"], c["hv"], c["B"])

    def run(c, p):
        prm = _Params(c["M"], (1.0,) if c["M"] == 1 else (0.95, 1.0))
        return ops.step_patch(p, c["dt"], prm, y_first=c["y_first"])

    serial = [mk(c) for c in cases]
    rs = [run(c, p) for c, p in zip(cases, serial)]
    for rep in range(3):
        threaded = [mk(c) for c in cases]
        with ThreadPoolExecutor(8) as ex:
            rt = list(ex.map(run, cases, threaded))
        for a, b, ra, rb in zip(serial, threaded, rs, rt):
            for f in ("h", "hu", "hv"):
                assert same(getattr(a, f), getattr(b, f)), (rep, f)
            assert ra.max_wave_speed == rb.max_wave_speed
            assert ra.hyperbolicity_fixes == rb.hyperbolicity_fixes
            assert ra.wet_prefix_repairs == rb.wet_prefix_repairs
            assert np.array_equal(ra.clipped_mass, rb.clipped_mass)


def _perturbed_c2(j, i, eps):
    from paper_1803_01450_b200 import problems
    pb = problems.config2(n_coarse_steps=1)
    fine = np.array(pb.bathy_levels[1], copy=True)
    fine[j, i] += eps
    pb.bathy_levels = [pb.bathy_levels[0], fine]
    return pb


def test_non_telescoping_bathymetry_raises_like_the_reference(oracle):
    """C2's fixed level-2 layout tiles fine cells [128, 384)^2: a fine
    bathymetry value perturbed by 1e-9 m under it breaks the ladder, and
    the device check raises the reference's AssertionError (coarsen.py:95-100)
    as the oracle does; the same perturbation outside every level-2 patch
    is never checked, so both accept it."""
    from paper_1803_01450_b200.driver import Simulation
    bad = _perturbed_c2(200, 300, 1e-9)
    with pytest.raises(AssertionError):
        oracle.Simulation(bad)
    with pytest.raises(AssertionError, match="telescope"):
        Simulation(bad)
    ok = _perturbed_c2(10, 20, 1e-9)
    oracle.Simulation(ok)
    Simulation(ok)


def test_check_bathymetry_consistency_shim():
    """ops.check_bathymetry_consistency (coarsen.py:79-100): exact block
    means pass, a 2e-12 deviation under a covered coarse cell raises, and a
    deviation within atol passes."""
    from paper_1803_01450_b200 import ops
    from paper_1803_01450_b200.problems import block_mean
    rng = np.random.default_rng(7)
    M = 1
    fb = rng.uniform(-6.0, -5.0, (16, 32))
    fine = HostPatch((8, 4, 39, 19), 0.5, 0.5, np.zeros((M, 20, 36)), np.zeros((M, 20, 36)),
                     np.zeros((M, 20, 36)), np.full((20, 36), -6.0))
    fine.bathy[2:-2, 2:-2] = fb
    cb = np.full((16, 28), -5.5)
    cb[2 + 2:2 + 10, 2 + 4:2 + 20] = block_mean(fb, 2, 2)
    coarse = HostPatch((0, 0, 23, 11), 1.0, 1.0, np.zeros((M, 16, 28)), np.zeros((M, 16, 28)),
                       np.zeros((M, 16, 28)), cb)
    ops.check_bathymetry_consistency(fine, [coarse], 2, 2)
    coarse.bathy[2 + 5, 2 + 9] += 2e-12
    with pytest.raises(AssertionError):
        ops.check_bathymetry_consistency(fine, [coarse], 2, 2)
    coarse.bathy[2 + 5, 2 + 9] -= 2e-12
    coarse.bathy[2 + 5, 2 + 9] += 0.5e-12
    ops.check_bathymetry_consistency(fine, [coarse], 2, 2)
    assert same(coarse.h, np.zeros((M, 16, 28)))
