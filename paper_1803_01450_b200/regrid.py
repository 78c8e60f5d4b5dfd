"""Host-side regrid rules (regrid.py:58-232 under /root/reference/pkg/src/mlamr).

Per-cell flag tests run on the device (``mlamr_flag_cells``); the
level-wide morphology (dilate/erode, mesh.py:116-141), the nesting mask
(regrid.nesting_allowed, regrid.py:185-211) and the recursive-bisection
clustering (regrid.cluster_flags, regrid.py:129-182; native C++ in
``csrc/host_cluster.cpp``) run on the host, as in the reference.  The
harness rules of SURVEY.md App. B (gradient and Bernoulli flags, the
max-patch chop) are here too.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .mesh import IndexBox, dilate, erode, paint


def cluster_boxes(flags: np.ndarray, efficiency_target: float, allowed=None) -> np.ndarray:
    """regrid.cluster_flags (regrid.py:129-182) in native C++; int32 [n, 4]."""
    f = np.ascontiguousarray(flags, dtype=np.uint8)
    ny, nx = f.shape
    a = None if allowed is None else np.ascontiguousarray(allowed, dtype=np.uint8)
    # every box holds a flagged cell: ny*nx boxes always fit (np.empty only
    # commits the pages that get written)
    cap = max(ny * nx, 1)
    while True:
        out = np.empty((cap, 4), dtype=np.int32)
        n = N.lib().mlamr_cluster_flags(f.ctypes.data, ny, nx, float(efficiency_target),
                                        None if a is None else a.ctypes.data, out.ctypes.data, cap)
        if n == -2:
            raise ValueError("flags outside the allowed region; clear them first")
        if n >= 0:
            return out[:n]
        cap *= 8


_SAT_HOST = {}
_SAT_DEV = {}


def cluster_boxes_device(flags_d, allowed_d, ny: int, nx: int, efficiency_target: float, stream):
    """regrid.cluster_flags from device-resident 0/1 maps: the summed-area
    tables are exact int32 sums built on the GPU (``mlamr_sat_u8``); only
    the bisection recursion runs on the host (native C++)."""
    import torch
    key = (ny, nx)
    if key not in _SAT_HOST:
        _SAT_HOST[key] = (torch.empty((ny + 1) * (nx + 1), dtype=torch.int32, pin_memory=True),
                          torch.empty((ny + 1) * (nx + 1), dtype=torch.int32, pin_memory=True))
    hf, hb = _SAT_HOST[key]
    dkey = (ny, nx, flags_d.device)
    if dkey not in _SAT_DEV:
        with torch.cuda.stream(stream):
            _SAT_DEV[dkey] = (torch.empty(2 * (ny + 1) * (nx + 1), dtype=torch.int32, device=flags_d.device),
                              torch.empty(((ny + 31) // 32) * nx, dtype=torch.int32, device=flags_d.device))
    sat, scratch = _SAT_DEV[dkey]
    n1 = (ny + 1) * (nx + 1)
    lib = N.lib()
    with torch.cuda.stream(stream):
        for k, (src, invert) in enumerate(((flags_d, 0), (allowed_d, 1))):
            N.check(lib.mlamr_sat_u8(src.data_ptr(), ny, nx, invert, sat[k * n1:].data_ptr(), scratch.data_ptr(),
                                     stream.cuda_stream), "mlamr_sat_u8")
        hf.copy_(sat[:n1], non_blocking=True)
        hb.copy_(sat[n1:], non_blocking=True)
    stream.synchronize()
    return _cluster_from_sat(hf, hb, ny, nx, efficiency_target)


def _cluster_from_sat(hf, hb, ny, nx, efficiency_target):
    cap = max(ny * nx, 1)   # one pass (see cluster_boxes)
    while True:
        out = np.empty((cap, 4), dtype=np.int32)
        n = N.lib().mlamr_cluster_sat(hf.data_ptr(), hb.data_ptr(), ny, nx, float(efficiency_target),
                                      out.ctypes.data, cap)
        if n >= 0:
            return out[:n]
        cap *= 8


def chop_boxes(boxes: np.ndarray, max_nx: int, max_ny: int, aligned: bool = False) -> np.ndarray:
    """:func:`chop` in native C++ over an int32 [n, 4] array."""
    b = np.ascontiguousarray(boxes, dtype=np.int32).reshape(-1, 4)
    if len(b) == 0:
        return b
    areas = (b[:, 2] - b[:, 0] + 1).astype(np.int64) * (b[:, 3] - b[:, 1] + 1)
    cap = int(areas.sum()) if max_nx * max_ny == 1 else int(
        (((b[:, 2] - b[:, 0]) // max_nx + 2) * ((b[:, 3] - b[:, 1]) // max_ny + 2)).sum())
    out = np.empty((cap, 4), dtype=np.int32)
    n = N.lib().mlamr_chop_boxes(b.ctypes.data, len(b), max_nx, max_ny, int(aligned), out.ctypes.data, cap)
    if n < 0:
        raise RuntimeError("chop overflow")
    return out[:n]


def cluster_flags(flags: np.ndarray, efficiency_target: float, allowed=None):
    """regrid.cluster_flags (regrid.py:129-182): list of IndexBox."""
    return [IndexBox(*map(int, r)) for r in cluster_boxes(flags, efficiency_target, allowed)]


def chop(boxes, max_nx: int, max_ny: int, aligned: bool = False):
    """Harness max-patch-size chop: each box is cut into
    tiles of at most max_nx x max_ny coarse cells -- from the box corner, or
    (``aligned``) at global multiples of the tile size, so that interior
    tiles of neighbouring boxes line up -- then re-sorted by (lo_j, lo_i)."""
    out = []
    for b in boxes:
        if aligned:
            js = list(range(b.lo_j - b.lo_j % max_ny + max_ny, b.hi_j + 1, max_ny))
            is_ = list(range(b.lo_i - b.lo_i % max_nx + max_nx, b.hi_i + 1, max_nx))
            jcuts = [b.lo_j] + js
            icuts = [b.lo_i] + is_
        else:
            jcuts = list(range(b.lo_j, b.hi_j + 1, max_ny))
            icuts = list(range(b.lo_i, b.hi_i + 1, max_nx))
        for a, j in enumerate(jcuts):
            j1 = (jcuts[a + 1] - 1) if a + 1 < len(jcuts) else b.hi_j
            for c, i in enumerate(icuts):
                i1 = (icuts[c + 1] - 1) if c + 1 < len(icuts) else b.hi_i
                out.append(IndexBox(i, j, i1, j1))
    return sorted(out, key=lambda b: (b.lo_j, b.lo_i))


def nesting_allowed(level_boxes: np.ndarray, ny: int, nx: int) -> np.ndarray:
    """Union of the level's patches eroded by one cell, boundary-exempt."""
    return erode(paint(level_boxes, ny, nx), 1)


def reference_flags(bits: np.ndarray, M: int, buffer_width: int) -> np.ndarray:
    """regrid.flag_cells (regrid.py:58-101) from the device's per-cell bits:
    amplitude flags, plus wet cells within ``buffer_width`` of a dry cell of
    the same layer, dilated by ``buffer_width``, restricted to covered cells."""
    covered = (bits & 0x80) != 0
    flags = (bits & 1) != 0
    for m in range(M):
        wet = (bits & (2 << m)) != 0
        flags |= wet & dilate(covered & ~wet, buffer_width)
    return dilate(flags, buffer_width) & covered
