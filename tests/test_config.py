"""Run files: parsing/validation like the reference's config.py, and the
scenario fields bit for bit against the arrays the reference's Scenario
produced for the same shelf setup (tests/golden/run_shelf_small.npz)."""

import os

import numpy as np
import pytest

from conftest import load_golden

HERE = os.path.dirname(os.path.abspath(__file__))
CFG = os.path.join(HERE, "configs", "shelf_small.cfg")


def test_problem_from_config_matches_reference_scenario():
    from paper_1803_01450_b200.config import parse_config, problem_from_config
    z = load_golden("run_shelf_small.npz")
    cfg = parse_config(CFG)
    pb = problem_from_config(cfg)
    assert pb.t_final == 0.3 and pb.frame_times == (0.0, 0.15, 0.3)
    assert pb.densities == (0.95, 1.0) and pb.ratios_t == [2, 2]
    for lev, nx, ny, dx, dy, rx, ry, rt in pb.level_specs():
        spec = z[f"L{lev}_spec"]
        assert (nx, ny) == (int(spec[0]), int(spec[1]))
        if lev < pb.num_levels:
            assert (rx, ry, rt) == tuple(int(v) for v in spec[2:5])
        assert (dx, dy) == tuple(float(v) for v in z[f"L{lev}_dxdy"])
        B = pb.bathy_levels[lev - 1]
        assert np.array_equal(B, z[f"L{lev}_bathy"][2:-2, 2:-2])
        h, hu, hv = pb.initial_state_box(lev, (0, 0, nx - 1, ny - 1))
        for name, a in (("h", h), ("hu", hu), ("hv", hv)):
            assert np.array_equal(a, z[f"L{lev}_{name}"][:, 2:-2, 2:-2]), (lev, name)


def _text(**over):
    base = open(CFG).read()
    for key, val in over.items():
        sec, k = key.split("__")
        lines = base.splitlines()
        out, in_sec, done = [], False, False
        for ln in lines:
            if ln.startswith("["):
                if in_sec and not done and val is not None:
                    out.append(f"{k} = {val}")
                    done = True
                in_sec = ln.strip() == f"[{sec}]"
            if in_sec and ln.split("=")[0].strip() == k:
                if val is not None:
                    out.append(f"{k} = {val}")
                done = True
                continue
            out.append(ln)
        if in_sec and not done and val is not None:
            out.append(f"{k} = {val}")
        base = "\n".join(out) + "\n"
    return base


@pytest.mark.parametrize("over,key", [
    ({"grid__nx": "2"}, "grid.nx"),
    ({"grid__refine_x": "2"}, "grid.refine_x"),
    ({"time__cfl": "1.5"}, "time.cfl"),
    ({"time__frame_times": "0.2, 0.1"}, "time.frame_times"),
    ({"physics__num_layers": "3"}, "physics.num_layers"),
    ({"scenario__eta_rest": "0.0"}, "scenario.eta_rest"),
    ({"scenario__eta_rest": "-0.6, 0.0"}, "scenario.eta_rest"),
    ({"boundaries__left": "periodic"}, "boundaries.left"),
    ({"amr__wave_tolerance": "1e-3, 2e-3, 3e-3"}, "amr.wave_tolerance"),
    ({"amr__bogus": "1"}, "amr.bogus"),
    ({"scenario__b_right": None}, "scenario"),
    ({"time__t_final": None}, "time.t_final"),
])
def test_config_errors_name_the_key(over, key):
    from paper_1803_01450_b200.config import ConfigError, parse_config_text
    with pytest.raises(ConfigError) as ei:
        parse_config_text(_text(**over))
    assert ei.value.key == key


def test_config_defaults_and_regions():
    from paper_1803_01450_b200.config import parse_config_text, problem_from_config
    cfg = parse_config_text(_text(time__frame_times=None, amr__wave_tolerance="5e-3",
                                  amr__allowed_regions="0.0, 2.0, 0.0, 1.0; 3.0, 4.0, 0.25, 0.5"))
    assert cfg.frame_times == (0.0, 0.3)
    assert cfg.wave_tolerance == (5e-3, 5e-3)
    pb = problem_from_config(cfg)
    m = pb.region_mask(1)
    assert m.shape == (16, 64) and m[:, :32].all() and not m[:, 33:48].any()
    assert m[4:8, 48:].all() and not m[:4, 48:].any()


def test_cli_reports_config_errors(tmp_path):
    import subprocess
    import sys
    bad = tmp_path / "bad.cfg"
    bad.write_text(_text(grid__nx="2"))
    root = os.path.dirname(HERE)
    r = subprocess.run([sys.executable, "-m", "paper_1803_01450_b200", "run", str(bad), "--out", str(tmp_path)],
                       capture_output=True, text=True, cwd=root, timeout=300)
    assert r.returncode == 2 and "grid.nx" in r.stderr
