"""Size-independent properties of the GPU path, mirroring the reference's
own physics/driver tests (tests/test_driver.py, tests/test_physics.py
under /root/reference/pkg): lake at rest through regrids, the mass
accounting identity, bitwise determinism, bitwise mirror symmetry, an
exact dam-break solution, the non-finite abort with its dump frame, the
stats round trip -- and determinism plus the mass identity on the full
C4 configuration."""

import numpy as np
import pytest

from cfg_util import write_cfg

pytestmark = pytest.mark.gpu


def _surfaces(h, B):
    return np.cumsum(h[::-1], axis=0)[::-1] + B[None]


def test_lake_at_rest_three_levels_with_regrids(tmp_path):
    """reference tests/test_driver.py:86-117: |eta_m - rest_m| < 1e-11 on wet
    cells after 40 coarse steps of a 3-level run that keeps regridding."""
    from paper_1803_01450_b200.config import problem_from_config
    from paper_1803_01450_b200.driver import Simulation
    path = write_cfg(tmp_path, grid={"nx": 40, "ny": 8, "max_levels": 3, "refine_x": "2, 2", "refine_y": "2, 2"},
                     time={"t_final": 1.0, "frame_times": "", "cfl": 0.6}, scenario={"wave_amplitude": 0.0})
    pb = problem_from_config(path)
    sim = Simulation(pb)
    for _ in range(40):
        sim.advance_coarse_step(sim.choose_dt())
    assert sim.levels.get(3) is not None and sim.levels[3].P > 0, "front band should stay refined"
    worst = 0.0
    for lev in sim.levels:
        for box, h, hu, hv, b in sim.patch_fields(lev):
            hi, bi = h[:, 2:-2, 2:-2], b[2:-2, 2:-2]
            eta = _surfaces(hi, bi)
            for m, rest in enumerate(pb.eta_rest):
                wet = hi[m] > pb.dry_tolerance
                if wet.any():
                    worst = max(worst, float(np.abs(eta[m][wet] - rest).max()))
    assert worst < 1e-11, worst


def test_mass_identity_and_drift(tmp_path):
    """reference tests/test_driver.py:120-132."""
    from paper_1803_01450_b200.config import problem_from_config
    from paper_1803_01450_b200.driver import run_simulation
    pb = problem_from_config(write_cfg(tmp_path, time={"t_final": 0.2}))
    st = run_simulation(pb, t_final=pb.t_final, frame_times=pb.frame_times)
    for m in range(2):
        reported = st.refine_delta[m] + st.derefine_delta[m] + st.sync_delta[m]
        residual = st.final_mass[m] - st.initial_mass[m] - reported
        assert abs(residual) <= 1e-12 * st.initial_mass[m], (m, residual)
        assert abs(st.mass_drift[m]) <= 1e-3 * st.initial_mass[m]


def test_runs_are_bit_identical(tmp_path):
    """reference tests/test_driver.py:135-146."""
    from paper_1803_01450_b200.config import problem_from_config
    from paper_1803_01450_b200.driver import run_simulation
    path = write_cfg(tmp_path)
    outs = []
    for tag in ("a", "b"):
        pb = problem_from_config(path)
        st = run_simulation(pb, out_dir=tmp_path / tag, t_final=pb.t_final, frame_times=pb.frame_times)
        outs.append((st.total_cell_updates, (tmp_path / tag / "frame0001.bin").read_bytes()))
    assert outs[0] == outs[1]


def _single_level(nx, ny, domain, M, B, ic, boundaries=None, cfl=0.6):
    from paper_1803_01450_b200.problems import WALLS, Problem
    pb = Problem(name="single", domain=domain, coarse_nx=nx, coarse_ny=ny, ratios_x=[], ratios_y=[],
                 ratios_t=[], num_layers=M, densities=(0.95, 1.0)[-M:] if M == 2 else (1.0,), gravity=1.0,
                 dry_tolerance=1e-3, eta_rest=(0.0, -0.6)[:M], boundaries=dict(boundaries or WALLS), cfl=cfl,
                 dt_max=1.0)
    pb.bathy_levels = [np.full((ny, nx), float(B))]
    pb.ic = ic
    return pb


def test_mirror_symmetric_state_stays_symmetric_bitwise():
    """reference tests/test_physics.py:139-151: an x-symmetric two-layer
    bump stays bitwise symmetric (hu antisymmetric) for 100 steps."""
    from paper_1803_01450_b200.driver import Simulation

    def ic(p, level, xc, yc, jj, ii, B):
        ny, nx = B.shape
        h = np.zeros((2, ny, nx))
        h[1] = np.maximum(-0.6 - B, 0.0)
        h[0] = np.maximum(0.0 - (B + h[1]), 0.0)
        h[0] = h[0] + (0.03 * np.exp(-(((xc - 1.0) / 0.2) ** 2)))[None, :]
        return h, np.zeros_like(h), np.zeros_like(h)

    sim = Simulation(_single_level(32, 8, (0.0, 2.0, 0.0, 0.5), 2, -1.0, ic))
    for _ in range(100):
        sim.advance_coarse_step(sim.choose_dt())
    (box, h, hu, hv, b), = sim.patch_fields(1)
    h, hu = h[:, 2:-2, 2:-2], hu[:, 2:-2, 2:-2]
    assert np.array_equal(h, h[:, :, ::-1])
    assert np.array_equal(hu, -hu[:, :, ::-1])
    assert np.abs(hu).max() > 0.0


def _exact_dam_break(hl, hr, g, xi):
    """Exact wet-wet shallow-water Riemann solution (u_l = u_r = 0) at
    similarity coordinates xi = x/t: star depth by bisection on the
    shock/rarefaction depth functions, then the wave fan."""
    def wave(h, hk):
        if h > hk:
            return (h - hk) * np.sqrt(0.5 * g * (h + hk) / (h * hk))
        return 2.0 * (np.sqrt(g * h) - np.sqrt(g * hk))

    lo, hi = 1e-12, max(hl, hr)
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if wave(mid, hl) + wave(mid, hr) > 0.0:
            hi = mid
        else:
            lo = mid
    hs = 0.5 * (lo + hi)
    us = 0.5 * (wave(hs, hr) - wave(hs, hl))
    al, ar, as_ = np.sqrt(g * hl), np.sqrt(g * hr), np.sqrt(g * hs)
    out = np.empty_like(xi)
    for k, s in enumerate(xi):
        if s <= us:
            if hs > hl:
                sp = -al * np.sqrt(0.5 * (hs + hl) * hs / hl ** 2)
                out[k] = hl if s < sp else hs
            elif s < -al:
                out[k] = hl
            elif s > us - as_:
                out[k] = hs
            else:
                out[k] = ((2.0 * al - s) / 3.0) ** 2 / g
        else:
            if hs > hr:
                sp = ar * np.sqrt(0.5 * (hs + hr) * hs / hr ** 2)
                out[k] = hr if s > sp else hs
            elif s > ar:
                out[k] = hr
            elif s < us + as_:
                out[k] = hs
            else:
                out[k] = ((2.0 * ar + s) / 3.0) ** 2 / g
    return out


def test_dam_break_against_exact_solution():
    """reference tests/test_physics.py:154-168: 400 cells on [-1.5, 1.5],
    depths 1 / 0.5, t = 0.5, relative L1 error < 2 %."""
    from paper_1803_01450_b200.driver import Simulation

    def ic(p, level, xc, yc, jj, ii, B):
        h = np.where(xc < 0.0, 1.0, 0.5)[None, None, :] * np.ones((1,) + B.shape)
        return h, np.zeros_like(h), np.zeros_like(h)

    open_x = {"left": "outflow", "right": "outflow", "bottom": "wall", "top": "wall"}
    pb = _single_level(400, 4, (-1.5, 1.5, 0.0, 0.03), 1, 0.0, ic, open_x)
    pb.eta_rest = (2.0,)
    sim = Simulation(pb)
    sim.run_until(0.5)
    assert sim.time == pytest.approx(0.5, abs=1e-12)
    (box, h, hu, hv, b), = sim.patch_fields(1)
    hn = h[0, 2:-2, 2:-2][0]
    dx = 3.0 / 400
    xc = -1.5 + (np.arange(400) + 0.5) * dx
    sub = (np.arange(16) + 0.5) / 16 - 0.5
    ref = np.array([_exact_dam_break(1.0, 0.5, 1.0, (x + sub * dx) / 0.5).mean() for x in xc])
    err = np.abs(hn - ref).sum() / np.abs(ref).sum()
    assert err < 0.02, err


def test_non_finite_state_aborts_and_dumps(tmp_path, monkeypatch):
    """reference tests/test_driver.py:157-182."""
    from paper_1803_01450_b200.config import problem_from_config
    from paper_1803_01450_b200.driver import RunStats, Simulation, run_simulation
    from paper_1803_01450_b200.errors import NumericalAbortError
    path = write_cfg(tmp_path)
    sim = Simulation(problem_from_config(path))
    pool = sim.levels[1]
    NX = int(pool.boxes[0, 2] - pool.boxes[0, 0] + 1) + 4
    pool.state[5 * NX + 5] = float("nan")
    with pytest.raises(NumericalAbortError):
        sim.advance_coarse_step(1e-3)

    orig = Simulation.advance_coarse_step

    def poisoned(self, dt):
        p = self.levels[1]
        p.state[5 * NX + 5] = float("nan")
        orig(self, dt)

    monkeypatch.setattr(Simulation, "advance_coarse_step", poisoned)
    pb = problem_from_config(path)
    with pytest.raises(NumericalAbortError):
        run_simulation(pb, out_dir=tmp_path / "dump", t_final=pb.t_final, frame_times=pb.frame_times)
    assert (tmp_path / "dump" / "abort.bin").exists()
    st = RunStats.from_json(tmp_path / "dump" / "stats.json")
    # the reference counts the step, then checks finiteness (driver.py:305-309)
    assert st.num_coarse_steps == 1


def test_stats_json_round_trip(tmp_path):
    from paper_1803_01450_b200.config import problem_from_config
    from paper_1803_01450_b200.driver import RunStats, run_simulation
    pb = problem_from_config(write_cfg(tmp_path))
    st = run_simulation(pb, out_dir=tmp_path / "o", t_final=pb.t_final, frame_times=pb.frame_times)
    back = RunStats.from_json(tmp_path / "o" / "stats.json")
    assert back.total_cell_updates == st.total_cell_updates
    assert back.cell_updates_per_level == st.cell_updates_per_level
    np.testing.assert_allclose(back.final_mass, st.final_mass)


def test_c4_full_size_determinism_and_mass_identity():
    """BASELINE config C4 at full size (512^2 level 1, ~35 M finest cells):
    two independent runs of two coarse steps write identical frames, and
    the mass accounting identity holds to 1e-12 of the mass."""
    from paper_1803_01450_b200 import frames as F
    from paper_1803_01450_b200 import problems
    from paper_1803_01450_b200.driver import Simulation
    digests = []
    for _ in range(2):
        sim = Simulation(problems.config4())
        for _k in range(2):
            sim.advance_coarse_step(sim.choose_dt())
        st = sim.finish()
        import hashlib
        digests.append(hashlib.sha256(F.frame_bytes(sim)).hexdigest())
        for m in range(2):
            reported = st.refine_delta[m] + st.derefine_delta[m] + st.sync_delta[m]
            residual = st.final_mass[m] - st.initial_mass[m] - reported
            assert abs(residual) <= 1e-12 * st.initial_mass[m], (m, residual)
        del sim
    assert digests[0] == digests[1]
