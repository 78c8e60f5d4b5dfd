"""Pin the oracle (oracle/) against the reference's own outputs.

The golden vectors were produced by running the reference (mlamr, numpy +
numba) on seeded inputs: tests/golden/make_golden.py.  Fields must match
bit for bit (up to the sign of zero); mass diagnostics, which the
reference sums pairwise, within 1e-12 relative.
"""

import numpy as np
import pytest

from conftest import load_golden, mismatch, same


def test_step_patch_golden(oracle):
    z = load_golden("step_cases.npz")
    n = int(z["ncases"])
    for k in range(n):
        c = lambda key: z[f"c{k}_{key}"]
        M, nx, ny = int(c("M")), int(c("nx")), int(c("ny"))
        dens = (1.0,) if M == 1 else (0.95, 1.0)
        prm = oracle.Params(M, dens, 1.0, 1e-3)
        spec = oracle.Spec(1, nx, ny, float(c("dx")), float(c("dy")))
        p = oracle.OPatch(spec, oracle.Box(0, 0, nx - 1, ny - 1), M)
        p.bathy[...] = c("B")
        for s in range(4):
            p.h[...] = c(f"s{s}_pre_h")
            p.hu[...] = c(f"s{s}_pre_hu")
            p.hv[...] = c(f"s{s}_pre_hv")
            dt = float(c(f"s{s}_dt"))
            assert oracle.stable_dt(p, prm, 0.6) == dt
            r = oracle.step_patch(p, dt, prm, y_first=bool(c(f"s{s}_yfirst")))
            for f in ("h", "hu", "hv"):
                got = getattr(p, f)
                assert same(got, c(f"s{s}_{f}")), (k, s, f, mismatch(got, c(f"s{s}_{f}")))
            assert r.max_wave_speed == float(c(f"s{s}_speed"))
            assert r.hyperbolicity_fixes == int(c(f"s{s}_fixes"))
            assert r.wet_prefix_repairs == int(c(f"s{s}_repairs"))
            np.testing.assert_allclose(r.clipped_mass, c(f"s{s}_clipped"), rtol=1e-12, atol=1e-15)
            np.testing.assert_allclose(r.mass_delta, c(f"s{s}_mass_delta"), rtol=1e-9, atol=1e-13)


def test_step_exercises_repairs_and_blend():
    z = load_golden("step_cases.npz")
    n = int(z["ncases"])
    fixes = sum(int(z[f"c{k}_s{s}_fixes"]) for k in range(n) for s in range(4))
    repairs = sum(int(z[f"c{k}_s{s}_repairs"]) for k in range(n) for s in range(4))
    assert fixes > 0 and repairs > 0


def test_cfl_violation_raises_before_update(oracle):
    z = load_golden("step_cases.npz")
    assert int(z["cfl_raised"]) == 1
    prm = oracle.Params(2, (0.95, 1.0), 1.0, 1e-3)
    p = oracle.OPatch(oracle.Spec(1, 8, 8, 1 / 8, 1 / 8), oracle.Box(0, 0, 7, 7), 2)
    p.bathy[...] = z["cfl_B"]
    p.h[...] = z["cfl_h"]
    p.hu[...] = z["cfl_hu"]
    p.hv[...] = z["cfl_hv"]
    with pytest.raises(oracle.CflViolation):
        oracle.step_patch(p, float(z["cfl_dt"]), prm)
    assert same(p.h, z["cfl_h"]) and same(p.hu, z["cfl_hu"])


def test_interpolate_state_golden(oracle):
    z = load_golden("interp_cases.npz")
    for k in range(int(z["ncases"])):
        c = lambda key: z[f"c{k}_{key}"]
        M = int(c("M"))
        cb = oracle.Box(*[int(v) for v in c("cbox")])
        fb = oracle.Box(*[int(v) for v in c("fbox")])
        cd = oracle.Coarse(cb, c("h"), c("hu"), c("hv"), c("B"), c("avail"))
        dens = tuple(np.linspace(0.9, 1.0, M)) if M > 1 else (1.0,)
        prm = oracle.Params(M, dens, 1.0, 1e-3)
        oh, ohu, ohv = oracle.interpolate_state(cd, fb, c("fb"), int(c("rx")), int(c("ry")), prm)
        assert same(oh, c("oh")), k
        assert same(ohu, c("ohu")), k
        assert same(ohv, c("ohv")), k


def test_block_mean_golden(oracle):
    z = load_golden("blockmean_cases.npz")
    for k in range(int(z["ncases"])):
        rx, ry = (int(v) for v in z[f"c{k}_r"])
        assert same(oracle.block_mean(z[f"c{k}_a"], rx, ry), z[f"c{k}_out"]), (rx, ry)


def test_cluster_flags_golden(oracle):
    z = load_golden("cluster_cases.npz")
    for k in range(int(z["ncases"])):
        allowed = z[f"c{k}_allowed"]
        allowed = None if allowed.size == 0 else allowed
        boxes = oracle.cluster_flags(z[f"c{k}_flags"], float(z[f"c{k}_eff"]), allowed)
        got = np.array([list(b) for b in boxes], dtype=np.int64).reshape(-1, 4)
        assert np.array_equal(got, z[f"c{k}_boxes"]), k
    assert np.array_equal(oracle.dilate(z["dilate_in"], 2), z["dilate_out"])
    assert np.array_equal(oracle.erode(z["dilate_in"], 1), z["erode_out"])


def _compare_hier(sim, z, prefix):
    for lev in range(1, sim.L + 1):
        boxes = np.array([list(p.box) for p in sim.patches[lev]], dtype=np.int64).reshape(-1, 4)
        assert np.array_equal(boxes, z[f"{prefix}L{lev}_boxes"]), (prefix, lev)
        for k, p in enumerate(sim.patches[lev]):
            jj, ii = p.inner
            for f in ("h", "hu", "hv"):
                ref = z[f"{prefix}L{lev}_p{k}_{f}"]
                got = getattr(p, f)
                assert same(got[:, jj, ii], ref[:, jj, ii]), (prefix, lev, k, f,
                                                              mismatch(got[:, jj, ii], ref[:, jj, ii]))
            assert same(p.bathy, z[f"{prefix}L{lev}_p{k}_bathy"]), (prefix, lev, k)


def test_driver_run_golden(oracle):
    """Whole subcycled run (regrid, fill, step, coarsen) of the reference's
    shelf_demo_small config: layouts and interiors bit-exact."""
    from shelf_problem import shelf_problem
    z = load_golden("run_shelf_small.npz")
    sim = oracle.Simulation(shelf_problem())
    _compare_hier(sim, z, "t0_")
    dts = z["dts"]
    for step in range(len(dts)):
        dt = sim.choose_dt()
        assert dt == float(dts[step])
        sim.advance_coarse_step(dt)
        if step == 1:
            _compare_hier(sim, z, "s2_")
    _compare_hier(sim, z, "final_")
    st = sim.stats
    assert st.total_cell_updates == int(z["stat_total_cell_updates"])
    assert st.num_regrids == int(z["stat_num_regrids"])
    assert st.hyperbolicity_warnings == int(z["stat_fixes"])
    assert st.wet_prefix_repairs == int(z["stat_repairs"])
    for key, mine in (("clipped", st.clipped_mass), ("refine_delta", st.refine_delta),
                      ("derefine_delta", st.derefine_delta), ("sync_delta", st.sync_delta)):
        np.testing.assert_allclose(mine, z[f"stat_{key}"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(sim.composite_mass(), z["final_mass"], rtol=1e-12)
    assert [sim.steps[l] for l in sorted(sim.steps)] == list(z["steps"])


def test_ghost_fill_blended_golden(oracle):
    """ghost.fill_ghosts through the driver's blended parent provider
    (driver.py:157-190): every ghost cell of every level-3 patch."""
    from shelf_problem import shelf_problem
    z = load_golden("run_shelf_small.npz")
    sim = oracle.Simulation(shelf_problem())
    for step in range(len(z["dts"])):
        sim.advance_coarse_step(sim.choose_dt())
    lev = 3
    # install the captured pre-fill state and the blended stash
    for k, p in enumerate(sim.patches[lev]):
        for f in ("h", "hu", "hv"):
            getattr(p, f)[...] = z[f"gf_before_L{lev}_p{k}_{f}"]
    parents = sim.patches[lev - 1]
    old = {}
    for k, p in enumerate(parents):
        for f in ("h", "hu", "hv"):
            getattr(p, f)[...] = z[f"gf_before_L{lev - 1}_p{k}_{f}"]
        key = f"gf_parent_{k}"
        old[id(p)] = (z[key + "_oh"], z[key + "_ohu"], z[key + "_ohv"])
    sim._stash[lev - 1] = (float(z["gf_t0"]), float(z["gf_dt"]), old)
    sim.fill_level_ghosts(lev, float(z["gf_t"]))
    for k, p in enumerate(sim.patches[lev]):
        for f in ("h", "hu", "hv"):
            ref = z[f"gf_after_L{lev}_p{k}_{f}"]
            assert same(getattr(p, f), ref), (k, f, mismatch(getattr(p, f), ref))
