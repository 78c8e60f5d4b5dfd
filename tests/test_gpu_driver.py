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


@pytest.mark.parametrize("name,steps", [("C1", 3), ("C2", 2)])
def test_config_run_matches_oracle(oracle, name, steps):
    from paper_1803_01450_b200 import problems
    from paper_1803_01450_b200.driver import Simulation
    pb = problems.CONFIGS[name]()
    gpu = Simulation(pb)
    cpu = oracle.Simulation(pb)
    assert compare_levels(gpu, cpu) == []
    for _ in range(steps):
        dt_c = cpu.choose_dt()
        dt_g = gpu.choose_dt()
        assert dt_c == dt_g
        cpu.apply_dynamic_rt(dt_c)
        gpu.apply_dynamic_rt(dt_g)
        cpu.advance_coarse_step(dt_c)
        gpu.advance_coarse_step(dt_g)
        assert compare_levels(gpu, cpu) == []
    sg = gpu.finish()
    assert sg.total_cell_updates == cpu.stats.total_cell_updates
    assert sg.num_regrids == cpu.stats.num_regrids
