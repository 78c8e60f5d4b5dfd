"""GPU parity of whole subcycled AMR runs (regrid + ghost fill + step +
coarsen, level-batched through the C-ABI) against the reference's golden
run and against the oracle."""

import numpy as np
import pytest

from conftest import load_golden, mismatch, same
from gpu_util import compare_levels

pytestmark = pytest.mark.gpu


def _compare_golden(sim, z, prefix):
    for lev in range(1, sim.L + 1):
        got = sim.patch_fields(lev)
        boxes = np.array([g[0] for g in got], dtype=np.int64).reshape(-1, 4)
        assert np.array_equal(boxes, z[f"{prefix}L{lev}_boxes"]), (prefix, lev)
        for k, (box, h, hu, hv, b) in enumerate(got):
            for f, arr in (("h", h), ("hu", hu), ("hv", hv)):
                ref = z[f"{prefix}L{lev}_p{k}_{f}"][:, 2:-2, 2:-2]
                assert same(arr[:, 2:-2, 2:-2], ref), (prefix, lev, k, f, mismatch(arr[:, 2:-2, 2:-2], ref))
            assert same(b, z[f"{prefix}L{lev}_p{k}_bathy"]), (prefix, lev, k)


def test_shelf_small_run_matches_reference():
    from shelf_problem import shelf_problem
    from paper_1803_01450_b200.driver import Simulation
    z = load_golden("run_shelf_small.npz")
    sim = Simulation(shelf_problem())
    _compare_golden(sim, z, "t0_")
    for step, dtref in enumerate(z["dts"]):
        dt = sim.choose_dt()
        assert dt == float(dtref)
        sim.advance_coarse_step(dt)
        if step == 1:
            _compare_golden(sim, z, "s2_")
    _compare_golden(sim, z, "final_")
    st = sim.finish()
    assert st.total_cell_updates == int(z["stat_total_cell_updates"])
    assert st.num_regrids == int(z["stat_num_regrids"])
    assert st.hyperbolicity_warnings == int(z["stat_fixes"])
    assert st.wet_prefix_repairs == int(z["stat_repairs"])
    for key, mine in (("clipped", st.clipped_mass), ("refine_delta", st.refine_delta),
                      ("derefine_delta", st.derefine_delta), ("sync_delta", st.sync_delta)):
        np.testing.assert_allclose(mine, z[f"stat_{key}"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(st.final_mass, z["final_mass"], rtol=1e-12)


def _variant(name):
    """Small but complete variants of the BASELINE configs: every code path
    (M=1/2/3, r=(4,1)/(4,4)/(4,2), gradient/Bernoulli/reference flags,
    dynamic r_t, chop, frequent regrids with refine + copy + derefine)."""
    from paper_1803_01450_b200 import problems
    if name == "C1":
        return problems.config1(), 3
    if name == "C2":
        return problems.config2(), 2
    if name == "C3":
        pb = problems.config3(nx0=32)
        pb.regrid_interval = 2
        return pb, 3
    if name == "C4":
        pb = problems.config4(nx0=64)
        pb.regrid_interval = 2
        return pb, 2
    if name == "C5":
        pb = problems.config5(nx0=64)
        pb.bernoulli = (0.05,)     # sparse flags: the layout changes every step
        return pb, 3
    raise KeyError(name)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_config_run_matches_oracle(oracle, name):
    from paper_1803_01450_b200.driver import Simulation
    pb, steps = _variant(name)
    gpu = Simulation(pb)
    cpu = oracle.Simulation(pb)
    assert compare_levels(gpu, cpu) == []
    for _ in range(steps):
        dt_c = cpu.choose_dt()
        dt_g = gpu.choose_dt()
        assert dt_c == dt_g
        cpu.apply_dynamic_rt(dt_c)
        gpu.apply_dynamic_rt(dt_g)
        assert [s.r_t for s in cpu.specs] == [s.r_t for s in gpu.specs]
        cpu.advance_coarse_step(dt_c)
        gpu.advance_coarse_step(dt_g)
        assert compare_levels(gpu, cpu) == []
    sg = gpu.finish()
    sc = cpu.stats
    assert sg.total_cell_updates == sc.total_cell_updates
    assert sg.num_regrids == sc.num_regrids
    assert sg.hyperbolicity_warnings == sc.hyperbolicity_warnings
    assert sg.wet_prefix_repairs == sc.wet_prefix_repairs
    # mass diagnostics are sums whose order differs (numpy pairwise vs tree
    # reductions); refine/derefine deltas are differences of ~1e14 m^3 sums,
    # so they are compared at 1e-12 of the mass scale
    mass = cpu.composite_mass()
    scale = float(np.abs(mass).sum())
    np.testing.assert_allclose(sg.clipped_mass, sc.clipped_mass, rtol=1e-9, atol=1e-12 * scale)
    for a, b in ((sg.refine_delta, sc.refine_delta), (sg.derefine_delta, sc.derefine_delta)):
        np.testing.assert_allclose(np.asarray(a, float), np.asarray(b, float), rtol=0, atol=1e-12 * scale)
    np.testing.assert_allclose(gpu.composite_mass(), mass, rtol=1e-12)


def test_shelf_small_with_separate_sibling_copy_matches_reference():
    """The separate sibling-copy fill of the finest level (instead of the
    default: the step reading sibling halo cells through the ghost plan)
    gives the same bits."""
    from shelf_problem import shelf_problem
    from paper_1803_01450_b200.driver import Simulation
    z = load_golden("run_shelf_small.npz")
    sim = Simulation(shelf_problem())
    sim.fuse_sibling_fill = False
    for dtref in z["dts"]:
        dt = sim.choose_dt()
        assert dt == float(dtref)
        sim.advance_coarse_step(dt)
    _compare_golden(sim, z, "final_")


@pytest.mark.parametrize("bathymetry", [False, True])
def test_snapshot_restore_continues_bit_identically(bathymetry):
    """Checkpoint/restore (the e2e path): a simulation restored from a
    pinned-host snapshot -- with or without the pools' bathymetry, which a
    restore otherwise re-derives on the device -- continues bit for bit
    like the original."""
    from paper_1803_01450_b200 import problems
    from paper_1803_01450_b200.driver import Simulation
    pb = problems.config4(nx0=64)
    pb.regrid_interval = 2
    a = Simulation(pb)
    for _ in range(2):
        a.advance_coarse_step(a.choose_dt())
    snap = a.snapshot(bathymetry=bathymetry)
    b = Simulation.restore(pb, snap)
    for _ in range(2):
        dt = a.choose_dt()
        assert b.choose_dt() == dt
        a.advance_coarse_step(dt)
        b.advance_coarse_step(dt)
    assert a.time == b.time and a.stats.total_cell_updates == b.stats.total_cell_updates
    # the snapshot is a deep copy: the two runs' counters are their own
    assert a.stats.cell_updates_per_level == b.stats.cell_updates_per_level
    assert a.stats.sync_delta == b.stats.sync_delta
    assert a.stats.cell_updates_per_level is not b.stats.cell_updates_per_level
    assert snap["stats"].cell_updates_per_level != a.stats.cell_updates_per_level
    for lev in range(1, a.L + 1):
        fa, fb = a.patch_fields(lev), b.patch_fields(lev)
        assert [x[0] for x in fa] == [x[0] for x in fb]
        for x, y in zip(fa, fb):
            for u, v in zip(x[1:4], y[1:4]):
                assert np.array_equal(u[:, 2:-2, 2:-2], v[:, 2:-2, 2:-2])
            assert np.array_equal(x[4], y[4])
    np.testing.assert_array_equal(a.composite_mass(), b.composite_mass())


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_walker_step_form_matches_oracle(oracle, name):
    """The line-walker form of K1 (csrc/step_walk.cuh, mlamr_set_step_form)
    is bit-identical to the oracle on the wide-tile configs."""
    from paper_1803_01450_b200 import _native as N
    from paper_1803_01450_b200.driver import Simulation
    prev = N.lib().mlamr_set_step_form(1)
    try:
        pb, steps = _variant(name)
        gpu = Simulation(pb)
        cpu = oracle.Simulation(pb)
        for _ in range(steps):
            dt = cpu.choose_dt()
            assert gpu.choose_dt() == dt
            cpu.apply_dynamic_rt(dt)
            gpu.apply_dynamic_rt(dt)
            cpu.advance_coarse_step(dt)
            gpu.advance_coarse_step(dt)
            assert compare_levels(gpu, cpu) == []
    finally:
        N.lib().mlamr_set_step_form(prev)


def _level1_composite(sim):
    """Level 1's interior cells on the full grid, whatever its patches."""
    s = sim.spec(1)
    out = None
    for box, h, hu, hv, _ in sim.patch_fields(1):
        if out is None:
            out = np.full((3, h.shape[0], s.ny, s.nx), np.nan)
        lo_i, lo_j, hi_i, hi_j = box
        for q, a in enumerate((h, hu, hv)):
            out[q, :, lo_j:hi_j + 1, lo_i:hi_i + 1] = a[:, 2:-2, 2:-2]
    return out


@pytest.mark.parametrize("name,tile", [("C2", 32), ("C3", 16), ("C4", 16), ("C5", 32)])
def test_tiled_level1_is_bit_identical(monkeypatch, name, tile):
    """Level 1 cut into aligned tiles (MLAMR_L1_TILE; what a sharded run
    spreads over the ranks) steps bit for bit like the reference's single
    level-1 patch (mesh.py:372-375; SURVEY.md App. C probe 4): same layouts
    and fields on the finer levels, same level-1 cells, same dt."""
    from paper_1803_01450_b200.driver import Simulation
    pb, steps = _variant(name)
    ref = Simulation(pb)
    monkeypatch.setenv("MLAMR_L1_TILE", str(tile))
    til = Simulation(pb)
    monkeypatch.delenv("MLAMR_L1_TILE")
    assert til.levels[1].P > 1 and ref.levels[1].P == 1
    for _ in range(steps):
        dt = ref.choose_dt()
        assert til.choose_dt() == dt
        for sim in (ref, til):
            sim.apply_dynamic_rt(dt)
            sim.advance_coarse_step(dt)
        assert np.array_equal(_level1_composite(ref), _level1_composite(til))
        for lev in range(2, ref.L + 1):
            fa, fb = ref.patch_fields(lev), til.patch_fields(lev)
            assert [x[0] for x in fa] == [x[0] for x in fb]
            for x, y in zip(fa, fb):
                for u, v in zip(x[1:4], y[1:4]):
                    assert np.array_equal(u[:, 2:-2, 2:-2], v[:, 2:-2, 2:-2])
