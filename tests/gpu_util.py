"""Helpers for the GPU parity tests."""

import numpy as np

from conftest import mismatch, same


class HostPatch:
    """Minimal stand-in for mlamr.mesh.Patch (mesh.py:144-232)."""

    def __init__(self, box, dx, dy, h, hu, hv, bathy, level=1):
        self.box = tuple(int(v) for v in box)
        self.dx = dx
        self.dy = dy
        self.h = np.array(h, dtype=np.float64)
        self.hu = np.array(hu, dtype=np.float64)
        self.hv = np.array(hv, dtype=np.float64)
        self.bathy = np.array(bathy, dtype=np.float64)
        self.level = level
        self.ghost_width = 2


def compare_levels(gpu_sim, oracle_sim, levels=None, fields=("h", "hu", "hv")):
    """Layouts bit-exact; interiors bit-exact (sign of zero aside)."""
    levels = levels or range(1, oracle_sim.L + 1)
    report = []
    for lev in levels:
        ops = oracle_sim.patches[lev]
        gps = gpu_sim.patch_fields(lev)
        assert [tuple(p.box) for p in ops] == [g[0] for g in gps], f"layout differs on level {lev}"
        for k, (p, g) in enumerate(zip(ops, gps)):
            jj, ii = p.inner
            for name, garr in zip(("h", "hu", "hv"), g[1:4]):
                if name not in fields:
                    continue
                a = getattr(p, name)[:, jj, ii]
                b = garr[:, 2:-2, 2:-2]
                if not same(a, b):
                    report.append((lev, k, name, mismatch(a, b), float(np.nanmax(np.abs(a - b)))))
    return report
