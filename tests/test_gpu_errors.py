"""Failure detection on the GPU path: the reference's error
semantics through the C-ABI status word."""

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


def test_driver_cfl_violation_raises_and_spares_the_patch():
    """A dt far above the stable one: CflViolationError, and the violating
    patches keep their pre-step interior (physics.py:342-347)."""
    from shelf_problem import shelf_problem
    from paper_1803_01450_b200.driver import Simulation
    from paper_1803_01450_b200.errors import CflViolationError
    sim = Simulation(shelf_problem())
    before = [f[1].copy() for f in sim.patch_fields(1)]
    dt = 20.0 * sim.choose_dt()
    with pytest.raises(CflViolationError):
        sim.advance_coarse_step(dt)
    after = sim.patch_fields(1)
    assert same(after[0][1][:, 2:-2, 2:-2], before[0][:, 2:-2, 2:-2])


def test_nonfinite_state_aborts():
    """A NaN injected into a level-2 interior: NumericalAbortError at the end
    of the coarse step (driver.py:286-297)."""
    import torch
    from shelf_problem import shelf_problem
    from paper_1803_01450_b200.driver import Simulation
    from paper_1803_01450_b200.errors import NumericalAbortError
    sim = Simulation(shelf_problem())
    pool = sim.levels[2]
    off = int(pool.offsets[0]) + 2 * (int(pool.boxes[0][2] - pool.boxes[0][0]) + 5) + 2
    pool.state[off] = float("nan")
    torch.cuda.synchronize()
    with pytest.raises(NumericalAbortError):
        sim.advance_coarse_step(sim.choose_dt())


def test_average_down_time_sync_error():
    from paper_1803_01450_b200 import ops
    from paper_1803_01450_b200.errors import TimeSyncError
    M = 2
    z = np.zeros((M, 8, 8))
    fine = HostPatch((0, 0, 3, 3), 0.5, 0.5, z + 1.0, z, z, np.zeros((8, 8)))
    coarse = HostPatch((0, 0, 1, 1), 1.0, 1.0, np.zeros((M, 6, 6)) + 1.0, np.zeros((M, 6, 6)),
                       np.zeros((M, 6, 6)), np.zeros((6, 6)))
    fine.time, coarse.time = 1.0, 1.5
    with pytest.raises(TimeSyncError):
        ops.average_down([fine], [coarse], 2, 2, _Params(M, (0.95, 1.0)))
    fine.time = 1.5
    ops.average_down([fine], [coarse], 2, 2, _Params(M, (0.95, 1.0)))
    assert np.all(coarse.h[:, 2:-2, 2:-2] == 1.0)


def test_refine_geometry_errors():
    from paper_1803_01450_b200 import ops
    from paper_1803_01450_b200.errors import GeometryError
    M = 2
    cd = ops.CoarseData((0, 0, 3, 3), np.ones((M, 4, 4)), np.zeros((M, 4, 4)), np.zeros((M, 4, 4)),
                        -np.ones((4, 4)), np.ones((4, 4), bool))
    fine = HostPatch((0, 0, 7, 7), 0.5, 0.5, np.zeros((M, 12, 12)), np.zeros((M, 12, 12)),
                     np.zeros((M, 12, 12)), -np.ones((12, 12)))
    prm = _Params(M, (0.95, 1.0))
    with pytest.raises(GeometryError):           # region outside the patch
        ops.refine_patch(cd, fine, 2, 2, prm, region=(4, 4, 9, 9))
    with pytest.raises(GeometryError):           # not ratio-aligned
        ops.refine_patch(cd, fine, 2, 2, prm, region=(1, 0, 4, 3))
    cd.avail[1, 1] = False
    with pytest.raises(GeometryError):           # incomplete coarse data
        ops.refine_patch(cd, fine, 2, 2, prm, region=(2, 2, 3, 3))
    with pytest.raises(GeometryError):           # parents outside the footprint
        ops.interpolate_state(cd, (0, 0, 9, 9), np.zeros((10, 10)), 2, 2, prm)


def test_empty_child_level_runs():
    """Flags that select nothing leave level 2 empty; the run proceeds on
    level 1 alone, like the reference with no refinement."""
    from paper_1803_01450_b200 import problems
    from paper_1803_01450_b200.driver import Simulation
    pb = problems.config2(n_coarse_steps=1)
    pb.fixed_layouts = {}
    pb.wave_tolerance = (1e9, 1e9)
    pb.buffer_width = 0
    pb.max_patch = None
    sim = Simulation(pb)
    assert sim.levels.get(2) is None or sim.levels[2].P == 0
    sim.advance_coarse_step(sim.choose_dt())
    assert sim.stats.total_cell_updates == 128 * 128


def test_nonfinite_check_reads_fused_sibling_ghosts_through_the_plan():
    """With the sibling fill fused into the finest level's step, the finite
    check (driver.py:286-297, isfinite over whole patch arrays) must see the
    sibling value a copy would have put in the ghost cell: a NaN in that
    sibling cell of the ghost-source buffer aborts, a NaN in the never-copied
    (stale) frame cell does not."""
    import torch
    from paper_1803_01450_b200 import problems
    from paper_1803_01450_b200.driver import Simulation
    from paper_1803_01450_b200.errors import NumericalAbortError
    sim = Simulation(problems.config2(n_coarse_steps=1))   # 8x8 tiling: siblings everywhere
    assert sim.fuse_sibling_fill
    sim.advance_coarse_step(sim.choose_dt())
    pool = sim.levels[sim.L]
    assert getattr(pool, "fused_frame", False) and not pool.ghosts_in_cur
    gbase, plan = (t.cpu().numpy() for t in pool.ghost_plan()[:2])
    g = int(np.flatnonzero(plan >= 0)[0])
    p = int(np.searchsorted(gbase, g, side="right") - 1)
    idx = g - int(gbase[p])
    b = pool.boxes[p]
    NX, NY = int(b[2] - b[0] + 5), int(b[3] - b[1] + 5)
    if idx < 2 * NX:
        J, I = divmod(idx, NX)
    elif idx < 4 * NX:
        J, I = divmod(idx - 2 * NX, NX)
        J += NY - 2
    else:
        q = idx - 4 * NX
        J, s = 2 + q // 4, q % 4
        I = (0, 1, NX - 2, NX - 1)[s]
    frame_cell = int(pool.offsets[p]) + J * NX + I
    # stale frame cell: not a ghost value of the fused path
    keep = pool.other[frame_cell].item()
    pool.other[frame_cell] = float("nan")
    sim.composite_mass()
    sim._sync_status("stale frame")
    pool.other[frame_cell] = keep
    # the sibling cell the copy would have read
    pool.other[int(plan[g])] = float("nan")
    torch.cuda.synchronize()
    sim.composite_mass()
    with pytest.raises(NumericalAbortError):
        sim._sync_status("sibling source")


def test_step_speed_is_nan_when_a_velocity_is_nan():
    """observed_max_speed (physics.py:261-278) takes numpy maxima, which
    propagate NaN: a NaN momentum in one wet interior cell makes that
    patch's observed speed NaN (canonical bits), the others stay finite."""
    import torch
    from paper_1803_01450_b200 import problems
    from paper_1803_01450_b200.driver import Simulation
    sim = Simulation(problems.config2(n_coarse_steps=1))
    sim.keep_step_speeds = True   # read the step's speeds afterwards
    lev = sim.L
    pool = sim.levels[lev]
    assert pool.P > 1
    sim.fill_level_ghosts(lev, sim.time)
    b = pool.boxes[0]
    NX = int(b[2] - b[0] + 5)
    cell = int(pool.offsets[0]) + 5 * NX + 7            # interior cell (5, 7) of patch 0
    M = sim.M
    assert pool.state[cell].item() > sim.pb.dry_tolerance   # top layer wet there
    pool.state[M * pool.FS + cell] = float("nan")          # hu of layer 0
    torch.cuda.synchronize()
    sim._step_patches(lev, 1e-3)
    bits = pool.speed_bits[:pool.P].cpu().numpy()
    assert bits[0] == 0x7FF8000000000000
    assert np.all((bits[1:] >= 0) & (bits[1:] < 0x7FF0000000000000))
