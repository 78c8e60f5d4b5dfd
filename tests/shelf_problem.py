"""Adapter: the reference's ``configs/shelf_demo_small.cfg`` as a harness
Problem, rebuilt from the arrays ``tests/golden/make_golden.py`` captured
from the reference Scenario (so no /root/reference access at run time)."""

import numpy as np

from paper_1803_01450_b200.problems import Problem

G = 2  # ghost width of the captured full-level arrays


class ShelfSmall(Problem):
    def __init__(self, z):
        super().__init__(
            name="shelf_demo_small", domain=(0.0, 4.0, 0.0, 1.0), coarse_nx=64, coarse_ny=16,
            ratios_x=[2, 2], ratios_y=[2, 2], ratios_t=[2, 2], num_layers=2,
            densities=(0.95, 1.0), gravity=1.0, dry_tolerance=1e-3, eta_rest=(0.0, -0.6),
            boundaries={"left": "outflow", "right": "outflow", "top": "wall", "bottom": "wall"},
            cfl=float(z["cfl"]), dt_max=float(z["dt_max"]), wave_tolerance=(2e-3, 4e-3),
            regrid_interval=2, buffer_width=2, efficiency_target=0.7,
        )
        self._z = z
        self._specs = []
        lev = 1
        while f"L{lev}_spec" in z:
            nx, ny, rx, ry, rt = (int(v) for v in z[f"L{lev}_spec"])
            dx, dy = (float(v) for v in z[f"L{lev}_dxdy"])
            self._specs.append((lev, nx, ny, dx, dy, rx, ry, rt))
            lev += 1
        self.bathy_levels = [z[f"L{l}_bathy"][G:-G, G:-G] for l in range(1, lev)]

    def level_specs(self):
        return list(self._specs)

    def _slice(self, key, level, box, layered):
        a = self._z[f"L{level}_{key}"]
        lo_i, lo_j, hi_i, hi_j = box
        sl = (slice(lo_j + G, hi_j + G + 1), slice(lo_i + G, hi_i + G + 1))
        return a[(slice(None),) + sl].copy() if layered else a[sl].copy()

    def initial_state_box(self, level, box):
        return tuple(self._slice(k, level, box, True) for k in ("h", "hu", "hv"))


def shelf_problem():
    from conftest import load_golden
    return ShelfSmall(load_golden("run_shelf_small.npz"))
