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


def _shelf_level_patches(z, prefix, lev):
    from gpu_util import HostPatch
    nx, ny = (int(v) for v in z[f"L{lev}_spec"][:2])
    dx, dy = (float(v) for v in z[f"L{lev}_dxdy"])
    out = []
    for k, b in enumerate(z[f"{prefix}L{lev}_boxes"]):
        p = HostPatch(b, dx, dy, z[f"{prefix}L{lev}_p{k}_h"], z[f"{prefix}L{lev}_p{k}_hu"],
                      z[f"{prefix}L{lev}_p{k}_hv"], z[f"{prefix}L{lev}_p{k}_bathy"], level=lev)
        p.time = 0.0
        out.append(p)
    return out, (0, 0, nx - 1, ny - 1)


def test_fill_ghosts_shim_blended_matches_reference():
    """ghost.fill_ghosts through a time-blended gather provider
    (driver.py:157-190) on the reference's captured level-3 state."""
    from paper_1803_01450_b200 import ops
    z = load_golden("run_shelf_small.npz")
    fine, lbox = _shelf_level_patches(z, "gf_before_", 3)
    parents, _ = _shelf_level_patches(z, "gf_before_", 2)
    stash = {id(p): (z[f"gf_parent_{k}_oh"], z[f"gf_parent_{k}_ohu"], z[f"gf_parent_{k}_ohv"])
             for k, p in enumerate(parents)}
    t, t0, dtp = float(z["gf_t"]), float(z["gf_t0"]), float(z["gf_dt"])
    theta = min(1.0, max(0.0, (t - t0) / dtp))
    prov = lambda box: ops.gather(parents, box, 2, blend=(theta, stash))
    bcs = {"left": "outflow", "right": "outflow", "top": "wall", "bottom": "wall"}
    prm = _Params(2, (0.95, 1.0))
    for p in fine:
        ops.fill_ghosts(p, fine, prov, bcs, lbox, 2, 2, prm)
    for k, p in enumerate(fine):
        for f in ("h", "hu", "hv"):
            ref = z[f"gf_after_L3_p{k}_{f}"]
            assert same(getattr(p, f), ref), (k, f, mismatch(getattr(p, f), ref))


def test_average_down_and_refine_shims_match_oracle(oracle):
    import copy
    from shelf_problem import shelf_problem
    from paper_1803_01450_b200 import ops
    sim = oracle.Simulation(shelf_problem())
    for _ in range(2):
        sim.advance_coarse_step(sim.choose_dt())
    prm = _Params(2, (0.95, 1.0))
    for lev in (2, 3):
        fine = sim.patches[lev]
        coarse_o = copy.deepcopy(sim.patches[lev - 1])
        coarse_g = copy.deepcopy(sim.patches[lev - 1])
        d_o = oracle.average_down(fine, coarse_o, 2, 2, sim.prm)
        d_g = ops.average_down(fine, coarse_g, 2, 2, prm)
        for a, b in zip(coarse_o, coarse_g):
            assert same(a.h, b.h) and same(a.hu, b.hu) and same(a.hv, b.hv), lev
        np.testing.assert_allclose(d_g, d_o, rtol=1e-9, atol=1e-12)
    # refine a whole level-3 patch from interior-only level-2 data
    p_o = copy.deepcopy(sim.patches[3][0])
    p_g = copy.deepcopy(sim.patches[3][0])
    run = p_o.box.coarse(2, 2).grow(1)
    c_o = oracle.gather(sim.patches[2], run, 2, include_ghosts=False)
    c_g = ops.gather(sim.patches[2], tuple(run), 2, include_ghosts=False)
    assert same(c_o.h, c_g.h) and np.array_equal(c_o.avail, c_g.avail)
    d_o = oracle.refine_patch(c_o, p_o, 2, 2, sim.prm)
    d_g = ops.refine_patch(c_g, p_g, 2, 2, prm)
    assert same(p_o.h, p_g.h) and same(p_o.hu, p_g.hu) and same(p_o.hv, p_g.hv)
    np.testing.assert_allclose(d_g, d_o, rtol=1e-12, atol=1e-12)


def test_average_down_block_means_match_reference_bitwise():
    """coarsen.block_mean (coarsen.py:21-27) as average_down evaluates it on
    the GPU, against the reference's own outputs: every ratio, including
    patches one coarse cell wide, whose r_y x r_x blocks numpy sums as one
    contiguous pairwise run (tests/golden/make_golden.py)."""
    from paper_1803_01450_b200 import ops
    z = load_golden("blockmean_cases.npz")
    for k in range(int(z["ncases"])):
        a = z[f"c{k}_a"]
        rx, ry = (int(v) for v in z[f"c{k}_r"])
        M, ny, nx = a.shape
        cny, cnx = ny // ry, nx // rx
        pad = lambda x: np.pad(x, ((0, 0), (2, 2), (2, 2)))  # noqa: E731
        fine = HostPatch((rx * 3, ry * 2, rx * 3 + nx - 1, ry * 2 + ny - 1), 1.0 / rx, 1.0 / ry,
                         pad(np.abs(a)), pad(a), pad(-a), np.zeros((ny + 4, nx + 4)))
        coarse = HostPatch((0, 0, cnx + 5, cny + 5), 1.0, 1.0, np.zeros((M, cny + 10, cnx + 10)),
                           np.zeros((M, cny + 10, cnx + 10)), np.zeros((M, cny + 10, cnx + 10)),
                           np.zeros((cny + 10, cnx + 10)))
        ops.average_down([fine], [coarse], rx, ry, _Params(M, (0.95, 1.0)), check_time=False)
        got = coarse.hu[:, 2 + 2:2 + 2 + cny, 2 + 3:2 + 3 + cnx]
        want = z[f"c{k}_out"]
        dry = coarse.h[:, 2 + 2:2 + 2 + cny, 2 + 3:2 + 3 + cnx] <= 1e-3
        assert same(got[~dry], want[~dry]), (k, rx, ry, a.shape, mismatch(got[~dry], want[~dry]))
