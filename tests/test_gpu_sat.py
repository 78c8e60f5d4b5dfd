"""mlamr_sat_u8: summed-area tables of 0/1 maps (the clustering's box
sums, regrid.cluster_flags) equal numpy's cumulative sums exactly."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ny,nx", [(1, 1), (1, 77), (77, 1), (31, 33), (64, 64), (257, 1000), (1000, 129)])
@pytest.mark.parametrize("invert", [0, 1])
def test_sat_equals_cumsum(ny, nx, invert):
    import torch
    from paper_1803_01450_b200 import _native as N
    rng = np.random.default_rng(ny * 1000 + nx + invert)
    m = (rng.random((ny, nx)) < 0.3).astype(np.uint8)
    md = torch.from_numpy(m).cuda()
    sat = torch.full(((ny + 1) * (nx + 1),), -7, dtype=torch.int32, device="cuda")
    scratch = torch.empty(((ny + 31) // 32) * nx, dtype=torch.int32, device="cuda")
    N.check(N.lib().mlamr_sat_u8(md.data_ptr(), ny, nx, invert, sat.data_ptr(), scratch.data_ptr(),
                                 torch.cuda.current_stream().cuda_stream), "sat")
    v = (1 - m.astype(np.int64)) if invert else m.astype(np.int64)
    ref = np.zeros((ny + 1, nx + 1), np.int64)
    ref[1:, 1:] = v.cumsum(0).cumsum(1)
    assert np.array_equal(sat.cpu().numpy().reshape(ny + 1, nx + 1), ref)


def test_device_bernoulli_flags_equal_host_rule():
    """mlamr_flags_bernoulli == the host rule (problems.bernoulli_flags,
    dilate, coverage, nesting) on a C5-shaped level, several steps."""
    from paper_1803_01450_b200 import problems
    from paper_1803_01450_b200.driver import Simulation
    from paper_1803_01450_b200.mesh import dilate, paint
    from paper_1803_01450_b200.regrid import nesting_allowed
    pb = problems.config5(nx0=64)
    pb.bernoulli = (0.05,)
    sim = Simulation(pb)
    s = sim.spec(1)
    for step in (0, 1, 7):
        sim.steps[1] = step
        flags, allowed = sim.flags_and_allowed(1)
        covered = paint(sim.levels[1].boxes, s.ny, s.nx)
        f = dilate(pb.bernoulli_flags(1, step), pb.flag_rule[2]) & covered
        al = nesting_allowed(sim.levels[1].boxes, s.ny, s.nx)
        assert np.array_equal(allowed, al)
        assert np.array_equal(flags, f & al)
        assert flags.any()


@pytest.mark.parametrize("name", ["C1", "C3"])
def test_device_gradient_flags_equal_host_rule(name):
    """mlamr_flags_gradient == the host rule (level surfaces,
    problems.gradient_flags_map, dilate, coverage, nesting)."""
    from paper_1803_01450_b200 import problems
    from paper_1803_01450_b200.driver import Simulation
    from paper_1803_01450_b200.mesh import dilate
    from paper_1803_01450_b200.problems import gradient_flags_map
    from paper_1803_01450_b200.regrid import nesting_allowed
    pb = problems.config1() if name == "C1" else problems.config3(nx0=32)
    sim = Simulation(pb)
    sim.advance_coarse_step(sim.choose_dt())
    _, tol, width, layers = pb.flag_rule
    checked = 0
    for lev in range(1, sim.L):
        if lev not in sim.levels or sim.levels[lev].P == 0:
            continue
        s = sim.spec(lev)
        flags, allowed = sim.flags_and_allowed(lev)
        eta, covered = sim.level_surfaces(lev, layers)
        f = dilate(gradient_flags_map(eta, covered, s.dx, s.dy, tol), width) & covered
        al = nesting_allowed(sim.levels[lev].boxes, s.ny, s.nx)
        assert np.array_equal(allowed, al), lev
        assert np.array_equal(flags, f & al), lev
        checked += int(flags.sum())
    assert checked > 0
