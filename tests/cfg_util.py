"""Run-file writer for tests (the reference's tests build theirs the same
way, tests/test_driver.py:10-36 there): a small two-layer shelf with
per-section overrides."""

BASE = {
    "domain": {"x_min": 0.0, "x_max": 4.0, "y_min": 0.0, "y_max": 1.0},
    "grid": {"nx": 32, "ny": 8, "max_levels": 2, "refine_x": "2", "refine_y": "2"},
    "time": {"t_final": 0.1, "frame_times": "0.0, 0.1", "cfl": 0.6},
    "physics": {"num_layers": 2, "density_ratio": 0.95},
    "scenario": {"bathymetry": "step", "step_x": 2.5, "b_left": -1.0, "b_right": -0.45,
                 "eta_rest": "0.0, -0.6", "wave_amplitude": 0.02, "wave_center": 2.25, "wave_width": 0.12},
    "boundaries": {"left": "wall", "right": "wall"},
    "amr": {"wave_tolerance": "2e-3, 4e-3"},
}


def write_cfg(tmp_path, **overrides) -> str:
    cfg = {k: dict(v) for k, v in BASE.items()}
    for section, kv in overrides.items():
        cfg.setdefault(section, {}).update(kv)
    lines = []
    for section, kv in cfg.items():
        lines.append(f"[{section}]")
        lines += [f"{k} = {v}" for k, v in kv.items()]
        lines.append("")
    path = tmp_path / "run.cfg"
    path.write_text("\n".join(lines))
    return str(path)
