"""ctypes binding of the handle-based patch-table runtime (csrc/patch_table.cu,
``mlamr_pt_*`` in include/mlamr_b200.h) -- what the reference would bind to
drive the GPU from its own host ``Patch`` arrays (numpy, mesh.py:158-232)
without torch: every argument is a host array or a scalar.

    pt = PatchTable(params_like, boundaries)
    pt.set_level(1, nx, ny, dx, dy, r_x, r_y, r_t)
    pt.upload(1, boxes, [p.h ...], [p.hu ...], [p.hv ...], [p.bathy ...])
    pt.fill_ghosts(1, t); pt.step(1, dt, y_first); h, hu, hv = pt.download(1)
"""

from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np

from . import _native as N
from .errors import CflViolationError, GeometryError, MlamrError, NumericalAbortError


def _ptrs(arrays: Sequence[np.ndarray]):
    arr = (ctypes.c_void_p * max(1, len(arrays)))()
    for k, a in enumerate(arrays):
        arr[k] = a.ctypes.data
    return arr


def _raise(rc: int, what: str) -> None:
    if rc == 0:
        return
    if rc == N.ST_CFL:
        raise CflViolationError(f"Courant number > 1 ({what})")
    if rc == N.ST_NONFINITE:
        raise NumericalAbortError(f"non-finite state ({what})")
    if rc == N.ST_GEOMETRY:
        raise GeometryError(f"coarse data footprint incomplete ({what})")
    raise MlamrError(f"{what} failed with code {rc}")


class PatchTable:
    """One device hierarchy managed by the native runtime."""

    def __init__(self, num_layers: int, densities, gravity: float, dry_tolerance: float, boundaries: dict,
                 stream=None):
        self.M = num_layers
        self.lib = N.lib()
        prm = N.make_params(num_layers, densities, gravity, dry_tolerance)
        self._bcs = N.bc_array(boundaries)
        self._h = self.lib.mlamr_pt_create(prm, ctypes.cast(self._bcs, ctypes.c_void_p), stream)
        if not self._h:
            raise MlamrError("mlamr_pt_create failed")
        self.boxes = {}

    def close(self) -> None:
        if self._h:
            self.lib.mlamr_pt_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    # -- hierarchy ------------------------------------------------------------------
    def set_level(self, level, nx, ny, dx, dy, r_x=1, r_y=1, r_t=1) -> None:
        _raise(self.lib.mlamr_pt_set_level(self._h, level, nx, ny, dx, dy, r_x, r_y, r_t), "set_level")

    def set_level_bathymetry(self, level: int, bathy: np.ndarray) -> None:
        b = np.ascontiguousarray(bathy, dtype=np.float64)
        _raise(self.lib.mlamr_pt_set_level_bathymetry(self._h, level, b.ctypes.data), "set_level_bathymetry")

    def upload(self, level: int, boxes, h, hu, hv, bathy=None) -> None:
        b = np.ascontiguousarray(np.asarray(boxes, dtype=np.int32).reshape(-1, 4))
        hs = [np.ascontiguousarray(a, dtype=np.float64) for a in h]
        hus = [np.ascontiguousarray(a, dtype=np.float64) for a in hu]
        hvs = [np.ascontiguousarray(a, dtype=np.float64) for a in hv]
        bs = [np.ascontiguousarray(a, dtype=np.float64) for a in bathy] if bathy is not None else None
        rc = self.lib.mlamr_pt_upload_patches(self._h, level, len(b), b.ctypes.data, _ptrs(hs), _ptrs(hus),
                                              _ptrs(hvs), _ptrs(bs) if bs is not None else None)
        _raise(rc, "upload_patches")
        self.boxes[level] = b

    def download(self, level: int):
        b = self.boxes[level]
        shp = [(self.M, int(r[3] - r[1] + 5), int(r[2] - r[0] + 5)) for r in b]
        h = [np.empty(s) for s in shp]
        hu = [np.empty(s) for s in shp]
        hv = [np.empty(s) for s in shp]
        _raise(self.lib.mlamr_pt_download(self._h, level, _ptrs(h), _ptrs(hu), _ptrs(hv)), "download")
        return h, hu, hv

    # -- operations -----------------------------------------------------------------
    def max_speed(self, level: int) -> np.ndarray:
        out = np.zeros(len(self.boxes.get(level, [])), np.float64)
        _raise(self.lib.mlamr_pt_max_speed(self._h, level, out.ctypes.data), "max_speed")
        return out

    def stash(self, level: int, t0: float, dt: float) -> None:
        _raise(self.lib.mlamr_pt_stash(self._h, level, t0, dt), "stash")

    def clear_stash(self, level: int) -> None:
        _raise(self.lib.mlamr_pt_clear_stash(self._h, level), "clear_stash")

    def fill_ghosts(self, level: int, t: float) -> None:
        _raise(self.lib.mlamr_pt_fill_ghosts(self._h, level, t), "fill_ghosts")

    def step(self, level: int, dt: float, y_first: bool = False) -> np.ndarray:
        """Returns [clipped depth per layer..., shear fixes, wet-prefix repairs]."""
        out = np.zeros(self.M + 2)
        bad = ctypes.c_int(-1)
        rc = self.lib.mlamr_pt_step_level(self._h, level, dt, int(bool(y_first)), out.ctypes.data,
                                          ctypes.addressof(bad))
        _raise(rc, f"step of level {level}, patch {bad.value}")
        return out

    def average_down(self, fine_level: int) -> None:
        _raise(self.lib.mlamr_pt_average_down(self._h, fine_level), "average_down")

    def regrid(self, level: int, new_boxes):
        b = np.ascontiguousarray(np.asarray(new_boxes, dtype=np.int32).reshape(-1, 4))
        ref = np.zeros(self.M)
        der = np.zeros(self.M)
        _raise(self.lib.mlamr_pt_regrid(self._h, level, len(b), b.ctypes.data, ref.ctypes.data, der.ctypes.data),
               "regrid")
        self.boxes[level] = b
        return ref, der

    def composite_mass(self) -> np.ndarray:
        out = np.zeros(self.M)
        _raise(self.lib.mlamr_pt_composite_mass(self._h, out.ctypes.data), "composite_mass")
        return out

    def check_finite(self) -> None:
        _raise(self.lib.mlamr_pt_check_finite(self._h), "check_finite")
