"""GPU parity of the per-patch drop-in operators (C-ABI, batch of one)
against the reference's golden vectors (tests/golden/)."""

import numpy as np
import pytest

from conftest import load_golden, mismatch, same
from gpu_util import HostPatch

pytestmark = pytest.mark.gpu


class _Params:
    def __init__(self, M, densities, g=1.0, tol=1e-3):
        self.num_layers = M
        self.densities = densities
        self.gravity = g
        self.dry_tolerance = tol


def test_step_patch_matches_reference_bitwise():
    from paper_1803_01450_b200 import ops
    z = load_golden("step_cases.npz")
    for k in range(int(z["ncases"])):
        c = lambda key: z[f"c{k}_{key}"]
        M, nx, ny = int(c("M")), int(c("nx")), int(c("ny"))
        prm = _Params(M, (1.0,) if M == 1 else (0.95, 1.0))
        for s in range(4):
            p = HostPatch((0, 0, nx - 1, ny - 1), float(c("dx")), float(c("dy")),
                          c(f"s{s}_pre_h"), c(f"s{s}_pre_hu"), c(f"s{s}_pre_hv"), c("B"))
            dt = float(c(f"s{s}_dt"))
            assert ops.stable_dt(p, prm, 0.6) == dt
            r = ops.step_patch(p, dt, prm, y_first=bool(c(f"s{s}_yfirst")))
            g = 2
            for f in ("h", "hu", "hv"):
                got = getattr(p, f)[:, g:-g, g:-g]
                ref = c(f"s{s}_{f}")[:, g:-g, g:-g]
                assert same(got, ref), (k, s, f, mismatch(got, ref))
            assert r.max_wave_speed == float(c(f"s{s}_speed"))
            assert r.hyperbolicity_fixes == int(c(f"s{s}_fixes"))
            assert r.wet_prefix_repairs == int(c(f"s{s}_repairs"))
            np.testing.assert_allclose(r.clipped_mass, c(f"s{s}_clipped"), rtol=1e-12, atol=1e-15)


def test_step_cfl_violation_leaves_patch_untouched():
    from paper_1803_01450_b200 import ops
    from paper_1803_01450_b200.errors import CflViolationError
    z = load_golden("step_cases.npz")
    p = HostPatch((0, 0, 7, 7), 1 / 8, 1 / 8, z["cfl_h"], z["cfl_hu"], z["cfl_hv"], z["cfl_B"])
    with pytest.raises(CflViolationError):
        ops.step_patch(p, float(z["cfl_dt"]), _Params(2, (0.95, 1.0)))
    assert same(p.h, z["cfl_h"])


def test_interpolate_state_matches_reference_bitwise():
    from paper_1803_01450_b200 import ops

    class CD:
        pass

    z = load_golden("interp_cases.npz")
    for k in range(int(z["ncases"])):
        c = lambda key: z[f"c{k}_{key}"]
        M = int(c("M"))
        cd = CD()
        cd.box = tuple(int(v) for v in c("cbox"))
        cd.h, cd.hu, cd.hv, cd.bathy, cd.avail = c("h"), c("hu"), c("hv"), c("B"), c("avail")
        dens = tuple(np.linspace(0.9, 1.0, M)) if M > 1 else (1.0,)
        oh, ohu, ohv = ops.interpolate_state(cd, tuple(int(v) for v in c("fbox")), c("fb"),
                                             int(c("rx")), int(c("ry")), _Params(M, dens))
        assert same(oh, c("oh")), (k, mismatch(oh, c("oh")))
        assert same(ohu, c("ohu")), k
        assert same(ohv, c("ohv")), k
