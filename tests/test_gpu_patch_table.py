"""The handle-based patch-table runtime (mlamr_pt_*, host arrays only)
drives the same kernels as the torch driver: a subcycled coarse step of
the shelf hierarchy and a regrid give the driver's bits."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pt_from_sim(sim):
    from paper_1803_01450_b200.patch_table import PatchTable
    pb = sim.pb
    pt = PatchTable(pb.num_layers, pb.densities, pb.gravity, pb.dry_tolerance, pb.boundaries)
    for lev in range(1, sim.L + 1):
        s = sim.spec(lev)
        pt.set_level(lev, s.nx, s.ny, s.dx, s.dy, s.r_x, s.r_y, s.r_t)
        pt.set_level_bathymetry(lev, pb.bathy_levels[lev - 1])
        if lev in sim.levels:
            f = sim.patch_fields(lev)
            pt.upload(lev, [x[0] for x in f], [x[1] for x in f], [x[2] for x in f], [x[3] for x in f],
                      [x[4] for x in f])
    return pt


def _advance_pt(pt, sim, steps, level, dt, t0):
    """The reference's recursion (driver.py:248-284) on the patch table."""
    pt.fill_ghosts(level, t0)
    has_child = level + 1 in sim.levels and sim.levels[level + 1].P > 0
    if has_child:
        pt.stash(level, t0, dt)
    pt.step(level, dt, y_first=bool(steps[level] % 2))
    steps[level] += 1
    if has_child:
        pt.fill_ghosts(level, t0 + dt)
        rt = sim.spec(level).r_t
        for k in range(rt):
            _advance_pt(pt, sim, steps, level + 1, dt / rt, t0 + k * dt / rt)
        pt.average_down(level + 1)
        pt.clear_stash(level)


def _same_interiors(pt, sim):
    for lev in sim.levels:
        h, hu, hv = pt.download(lev)
        for k, (box, sh, shu, shv, sb) in enumerate(sim.patch_fields(lev)):
            for a, b in ((h[k], sh), (hu[k], shu), (hv[k], shv)):
                assert np.array_equal(a[:, 2:-2, 2:-2].view(np.int64), b[:, 2:-2, 2:-2].view(np.int64)), (lev, k)


def test_patch_table_coarse_steps_match_driver():
    from shelf_problem import shelf_problem
    from paper_1803_01450_b200.driver import Simulation
    sim = Simulation(shelf_problem())
    sim.pb.regrid_interval = 10 ** 9
    sim.steps = {lv: 1 for lv in sim.steps}        # no regrid: both sides keep the layout
    pt = _pt_from_sim(sim)
    steps = dict(sim.steps)
    for _ in range(2):
        dt = sim.choose_dt()
        speeds = pt.max_speed(1)
        s1 = sim.spec(1)
        dt_pt = min(sim.pb.dt_max, sim.pb.cfl * min(s1.dx, s1.dy) / speeds.max())
        assert dt_pt == dt
        t0 = sim.time
        sim.advance_coarse_step(dt)
        _advance_pt(pt, sim, steps, 1, dt, t0)
        _same_interiors(pt, sim)
    np.testing.assert_allclose(pt.composite_mass(), sim.composite_mass(), rtol=1e-12)
    pt.check_finite()
    pt.close()


def test_patch_table_regrid_matches_driver():
    """A regrid of the finest level to new boxes (some kept, some new, some
    dropped): copied cells, refined cells and the mass deltas."""
    from shelf_problem import shelf_problem
    from paper_1803_01450_b200.driver import Simulation
    sim = Simulation(shelf_problem())
    sim.advance_coarse_step(sim.choose_dt())
    pt = _pt_from_sim(sim)
    L = sim.L
    s = sim.spec(L - 1)
    old = sim.levels[L].boxes
    # new coarse boxes: the old footprints shifted by one coarse cell in x
    cb = np.stack([old[:, 0] // s.r_x + 1, old[:, 1] // s.r_y, (old[:, 2] + 1) // s.r_x,
                   (old[:, 3] + 1) // s.r_y - 1], 1)
    cb[:, 2] = np.minimum(cb[:, 2], s.nx - 1)
    nb = np.stack([cb[:, 0] * s.r_x, cb[:, 1] * s.r_y, (cb[:, 2] + 1) * s.r_x - 1, (cb[:, 3] + 1) * s.r_y - 1], 1)
    d0 = sim.delta_acc.cpu().numpy().copy()
    sim._cluster_level = lambda level: cb            # inject the layout into the driver's rebuild
    assert sim._rebuild(L - 1)
    d1 = sim.delta_acc.cpu().numpy()
    ref, der = pt.regrid(L, nb)
    assert np.array_equal(np.asarray(sim.levels[L].boxes), nb)
    _same_interiors(pt, sim)
    np.testing.assert_allclose(ref, d1[0] - d0[0], rtol=1e-9, atol=1e-14)
    np.testing.assert_allclose(der, d1[1] - d0[1], rtol=1e-9, atol=1e-14)
    pt.close()
