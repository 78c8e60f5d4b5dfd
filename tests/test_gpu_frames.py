"""Frames written from the device pools (mlamr_pack_frame) are the bytes
the reference writes for the same run: shelf_demo_small at t=0 and after
two coarse steps, binary and text."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _diff_report(F, mine: bytes, ref: bytes):
    a, b = F.parse_frame(mine), F.parse_frame(ref)
    bad = []
    for k, (p, q) in enumerate(zip(a.patches, b.patches)):
        for f in ("bathy", "h", "hu", "hv"):
            x, y = getattr(p, f), getattr(q, f)
            if x.shape != y.shape or not np.array_equal(x.view(np.int64), y.view(np.int64)):
                bad.append((k, f))
    return bad


def test_device_frames_equal_reference_frames():
    from shelf_problem import shelf_problem
    from paper_1803_01450_b200 import frames as F
    from paper_1803_01450_b200.driver import Simulation
    z = load_golden("frames_shelf_small.npz")
    sim = Simulation(shelf_problem())
    for tag in ("t0", "s2"):
        if tag == "s2":
            for dtref in z["dts"]:
                dt = sim.choose_dt()
                assert dt == float(dtref)
                sim.advance_coarse_step(dt)
        for text in (False, True):
            ref = z[f"{tag}_{'txt' if text else 'bin'}"].tobytes()
            mine = F.frame_bytes(sim, text_mode=text)
            assert mine == ref, (tag, text, len(mine), len(ref), _diff_report(F, mine, ref))


def test_write_frame_and_compare(tmp_path):
    from shelf_problem import shelf_problem
    from paper_1803_01450_b200 import frames as F
    from paper_1803_01450_b200.driver import Simulation
    sim = Simulation(shelf_problem())
    F.write_frame(sim, tmp_path / "a.bin")
    sim.advance_coarse_step(sim.choose_dt())
    F.write_frame(sim, tmp_path / "b.bin")
    a, b = F.read_frame(tmp_path / "a.bin"), F.read_frame(tmp_path / "b.bin")
    assert a.time == 0.0 and b.time > 0.0
    assert F.l1_diff(a, b)["eta_1_linf"] > 0.0


def test_run_simulation_frames_and_stats_match_reference(tmp_path):
    """run_simulation to t_final with the config's frame times (dt clipped
    onto every frame time): frame files identical to the reference's, and
    the same stats.json counters."""
    import json
    from shelf_problem import shelf_problem
    from paper_1803_01450_b200.driver import run_simulation
    z = load_golden("frames_shelf_small.npz")
    st = run_simulation(shelf_problem(), out_dir=tmp_path, t_final=float(z["run_t_final"]),
                        frame_times=[float(t) for t in z["run_frame_times"]])
    for k in range(len(z["run_frame_times"])):
        mine = (tmp_path / f"frame{k:04d}.bin").read_bytes()
        assert mine == z[f"run_frame{k}"].tobytes(), k
    ref = json.loads(z["run_stats_json"].tobytes())
    got = json.loads((tmp_path / "stats.json").read_text())
    for key in ("total_cell_updates", "num_coarse_steps", "num_regrids", "hyperbolicity_warnings",
                "wet_prefix_repairs", "cell_updates_per_level", "amr_enabled", "workers"):
        assert got[key] == ref[key], key
    for key in ("initial_mass", "final_mass", "mass_drift", "refine_delta", "derefine_delta", "sync_delta",
                "clipped_mass"):
        np.testing.assert_allclose(got[key], ref[key], rtol=1e-9, atol=1e-12, err_msg=key)
    assert st.wall_time > 0.0


def test_run_file_to_reference_frames(tmp_path):
    """A run file through config.problem_from_config (the reference's
    Scenario, no captured arrays) reproduces the reference's run frames."""
    import os
    from paper_1803_01450_b200.config import problem_from_config
    from paper_1803_01450_b200.driver import run_simulation
    z = load_golden("frames_shelf_small.npz")
    pb = problem_from_config(os.path.join(os.path.dirname(__file__), "configs", "shelf_small.cfg"))
    run_simulation(pb, out_dir=tmp_path, t_final=pb.t_final, frame_times=pb.frame_times)
    for k in range(len(pb.frame_times)):
        assert (tmp_path / f"frame{k:04d}.bin").read_bytes() == z[f"run_frame{k}"].tobytes(), k


def test_cli_run_and_compare(tmp_path):
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cfg = os.path.join(root, "tests", "configs", "shelf_small.cfg")
    r = subprocess.run([sys.executable, "-m", "paper_1803_01450_b200", "run", cfg, "--out", str(tmp_path)],
                       capture_output=True, text=True, cwd=root, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert (tmp_path / "stats.json").exists() and (tmp_path / "frame0002.bin").exists()
    r = subprocess.run([sys.executable, "-m", "paper_1803_01450_b200", "compare", str(tmp_path / "frame0000.bin"),
                        str(tmp_path / "frame0002.bin"), "--norm", "all"], capture_output=True, text=True,
                       cwd=root, timeout=300)
    assert r.returncode == 0 and "eta_1_l1" in r.stdout and "h_2_linf" in r.stdout, r.stdout + r.stderr


def test_uniform_run_matches_reference_no_amr(tmp_path):
    """The reference's --no-amr run (one level at the finest resolution)."""
    import json
    import os
    from paper_1803_01450_b200.config import problem_from_config
    from paper_1803_01450_b200.driver import run_simulation
    z = load_golden("frames_shelf_small.npz")
    pb = problem_from_config(os.path.join(os.path.dirname(__file__), "configs", "shelf_small.cfg"),
                             uniform_fine=True)
    assert pb.num_levels == 1 and (pb.coarse_nx, pb.coarse_ny) == (256, 64)
    run_simulation(pb, out_dir=tmp_path, t_final=pb.t_final, frame_times=pb.frame_times)
    last = len(pb.frame_times) - 1
    assert (tmp_path / f"frame{last:04d}.bin").read_bytes() == z["uniform_frame_last"].tobytes()
    ref = json.loads(z["uniform_stats_json"].tobytes())
    got = json.loads((tmp_path / "stats.json").read_text())
    for key in ("total_cell_updates", "num_coarse_steps", "num_regrids", "amr_enabled", "cell_updates_per_level"):
        assert got[key] == ref[key], key
