"""ORACLE — test infrastructure only (never imported by the product path).

CPU restatement of the reference's multilayer-AMR hot path
(arxiv/paper_1803_01450, package ``mlamr``; paths below are relative to
``/root/reference/pkg/src/mlamr/``).  The arithmetic lives in
``orc_kernels.c`` (compiled with ``-ffp-contract=off``); this module
restates the orchestration around it: gathering coarse data, ghost bands,
boundary conditions, refinement/coarsening bookkeeping, regridding and the
subcycled level recursion.

Pinned against the reference itself: ``tests/golden/make_golden.py`` runs
the reference on seeded inputs in the build container and commits the
outputs; ``tests/test_oracle_golden.py`` checks this module against them.

Allowed importers: ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``
(cpu_baseline leg and ``--impl reference``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field, replace
from typing import Callable, NamedTuple, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liborc.so")
_lib = None

GHOST = 2
_dp = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)


def build() -> str:
    """Compile the C restatement (make in oracle/)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_step_patch.restype = ctypes.c_int
        L.orc_step_patch.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            _dp, _dp, _dp, _dp,
            ctypes.c_double, ctypes.c_double, ctypes.c_double,
            ctypes.c_double, ctypes.c_double, _dp, ctypes.c_int,
            ctypes.c_void_p,
        ]
        L.orc_observed_max_speed.restype = ctypes.c_double
        L.orc_observed_max_speed.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            _dp, _dp, _dp, ctypes.c_double, ctypes.c_double,
        ]
        L.orc_interpolate_state.restype = ctypes.c_int
        L.orc_interpolate_state.argtypes = [
            ctypes.c_int, _dp, _dp, _dp, _dp, _u8p,
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            _dp, ctypes.c_long, ctypes.c_int, ctypes.c_int, ctypes.c_double,
            _dp, _dp, _dp, ctypes.c_long, ctypes.c_long,
        ]
        L.orc_block_mean.restype = None
        L.orc_block_mean.argtypes = [
            _dp, ctypes.c_long, ctypes.c_int, ctypes.c_int,
            ctypes.c_int, ctypes.c_int, _dp, ctypes.c_long,
        ]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


class _StepRes(ctypes.Structure):
    _fields_ = [
        ("max_wave_speed", ctypes.c_double),
        ("mass_before", ctypes.c_double * 8),
        ("mass_after", ctypes.c_double * 8),
        ("clipped", ctypes.c_double * 8),
        ("cells_updated", ctypes.c_int64),
        ("fixes", ctypes.c_int64),
        ("repairs", ctypes.c_int64),
    ]


# --------------------------------------------------------------------------
# errors (errors.py:4-37)
# --------------------------------------------------------------------------
class OracleError(Exception):
    pass


class CflViolation(OracleError):
    pass


class GeometryFault(OracleError):
    pass


class TimeSyncFault(OracleError):
    pass


class NumericalAbort(OracleError):
    pass


# --------------------------------------------------------------------------
# geometry (mesh.py:23-113): inclusive index boxes as plain tuples
# --------------------------------------------------------------------------
class Box(NamedTuple):
    lo_i: int
    lo_j: int
    hi_i: int
    hi_j: int

    @property
    def nx(self):
        return self.hi_i - self.lo_i + 1

    @property
    def ny(self):
        return self.hi_j - self.lo_j + 1

    def meet(self, o: "Box") -> Optional["Box"]:
        a, b = max(self.lo_i, o.lo_i), max(self.lo_j, o.lo_j)
        c, d = min(self.hi_i, o.hi_i), min(self.hi_j, o.hi_j)
        if c < a or d < b:
            return None
        return Box(a, b, c, d)

    def grow(self, w: int) -> "Box":
        return Box(self.lo_i - w, self.lo_j - w, self.hi_i + w, self.hi_j + w)

    def covers(self, o: "Box") -> bool:
        return (self.lo_i <= o.lo_i and self.lo_j <= o.lo_j
                and o.hi_i <= self.hi_i and o.hi_j <= self.hi_j)

    def fine(self, rx: int, ry: int) -> "Box":
        return Box(self.lo_i * rx, self.lo_j * ry,
                   (self.hi_i + 1) * rx - 1, (self.hi_j + 1) * ry - 1)

    def coarse(self, rx: int, ry: int) -> "Box":
        if (self.lo_i % rx or self.lo_j % ry or (self.hi_i + 1) % rx
                or (self.hi_j + 1) % ry):
            raise GeometryFault(f"{self} not aligned to ({rx},{ry})")
        return Box(self.lo_i // rx, self.lo_j // ry,
                   (self.hi_i + 1) // rx - 1, (self.hi_j + 1) // ry - 1)


@dataclass(frozen=True)
class Spec:
    """One level of the ladder (mesh.py:23-38)."""
    level: int
    nx: int
    ny: int
    dx: float
    dy: float
    r_x: int = 1
    r_y: int = 1
    r_t: int = 1


@dataclass(frozen=True)
class Params:
    """state.LayerParams (state.py:19-53)."""
    M: int
    densities: tuple
    g: float
    tol: float = 1e-3

    @property
    def ratio(self) -> float:
        return self.densities[0] / self.densities[1]


class OPatch:
    """mesh.Patch (mesh.py:144-232): arrays [layer, j, i] with a 2-cell frame."""

    def __init__(self, spec: Spec, box: Box, M: int):
        self.spec = spec
        self.level = spec.level
        self.box = box
        self.time = 0.0
        NY, NX = box.ny + 2 * GHOST, box.nx + 2 * GHOST
        self.h = np.zeros((M, NY, NX))
        self.hu = np.zeros((M, NY, NX))
        self.hv = np.zeros((M, NY, NX))
        self.bathy = np.zeros((NY, NX))

    @property
    def full(self) -> Box:
        return self.box.grow(GHOST)

    def sl(self, b: Box):
        """Local slices of a global sub-box (may reach into the frame)."""
        fb = self.full
        if not fb.covers(b):
            raise ValueError(f"{b} outside {fb}")
        j0 = b.lo_j - fb.lo_j
        i0 = b.lo_i - fb.lo_i
        return slice(j0, j0 + b.ny), slice(i0, i0 + b.nx)

    @property
    def inner(self):
        return self.sl(self.box)


class BoxIndex:
    """Bucket grid over a patch list, keyed by every patch's frame (box grown
    by the ghost width).  ``query(box)`` returns, in list order, the patches
    whose frame meets ``box``: a superset of every interior or frame overlap
    the reference's O(P) scans find (ghost.py:58-84, :186-196; regrid.py:311-323,
    :334-348; coarsen.py:46-75, :79-100).  The scans below then run unchanged
    over the candidates, so their order and arithmetic are the reference's;
    the index only skips patches that cannot meet the box (test
    infrastructure: it makes the oracle reach the BASELINE sizes)."""

    S = 16

    def __init__(self, patches):
        self.patches = patches
        self.n = len(patches)
        self.buckets = {}
        S = self.S
        for k, p in enumerate(patches):
            f = p.box.grow(GHOST)
            for bj in range(f.lo_j // S, f.hi_j // S + 1):
                for bi in range(f.lo_i // S, f.hi_i // S + 1):
                    self.buckets.setdefault((bj, bi), []).append(k)

    def query(self, box: "Box"):
        S = self.S
        ks = set()
        for bj in range(box.lo_j // S, box.hi_j // S + 1):
            for bi in range(box.lo_i // S, box.hi_i // S + 1):
                got = self.buckets.get((bj, bi))
                if got:
                    ks.update(got)
        return [self.patches[k] for k in sorted(ks)]


# --------------------------------------------------------------------------
# physics (physics.py:261-386)
# --------------------------------------------------------------------------
def observed_max_speed(p: OPatch, prm: Params) -> float:
    M, NY, NX = p.h.shape
    return lib().orc_observed_max_speed(M, NY, NX, GHOST, _p(p.h), _p(p.hu), _p(p.hv),
                                        prm.g, prm.tol)


def stable_dt(p: OPatch, prm: Params, cfl: float, dt_max: float = 1.0) -> float:
    s = observed_max_speed(p, prm)
    if s <= 0.0:
        return dt_max
    return min(dt_max, cfl * min(p.spec.dx, p.spec.dy) / s)


@dataclass
class StepOut:
    max_wave_speed: float
    cells_updated: int
    mass_delta: np.ndarray
    hyperbolicity_fixes: int
    wet_prefix_repairs: int
    clipped_mass: np.ndarray


def step_patch(p: OPatch, dt: float, prm: Params, y_first: bool = False) -> StepOut:
    M, NY, NX = p.h.shape
    rho = np.ascontiguousarray(prm.densities, dtype=np.float64)
    res = _StepRes()
    st = lib().orc_step_patch(M, NY, NX, GHOST, _p(p.h), _p(p.hu), _p(p.hv), _p(p.bathy),
                              p.spec.dx, p.spec.dy, dt, prm.g, prm.tol, _p(rho),
                              int(bool(y_first)), ctypes.byref(res))
    if st == 3:
        c = res.max_wave_speed * dt / min(p.spec.dx, p.spec.dy)
        raise CflViolation(f"Courant number {c:.3f} > 1 on level {p.level} patch {p.box}")
    if st != 0:
        raise OracleError(f"orc_step_patch status {st}")
    return StepOut(
        max_wave_speed=res.max_wave_speed,
        cells_updated=int(res.cells_updated),
        mass_delta=np.array([res.mass_after[m] - res.mass_before[m] for m in range(M)]),
        hyperbolicity_fixes=int(res.fixes),
        wet_prefix_repairs=int(res.repairs),
        clipped_mass=np.array([res.clipped[m] for m in range(M)]),
    )


# --------------------------------------------------------------------------
# coarse data and interpolation (refine.py:50-239, ghost.py:29-86)
# --------------------------------------------------------------------------
@dataclass
class Coarse:
    box: Box
    h: np.ndarray
    hu: np.ndarray
    hv: np.ndarray
    bathy: np.ndarray
    avail: np.ndarray


def gather(patches, box: Box, M: int, blend=None, include_ghosts: bool = True,
           index: Optional[BoxIndex] = None) -> Coarse:
    """ghost.gather (ghost.py:29-86): interiors first; then, as a fallback,
    ghost frames in list order with the first provider winning.  ``index``
    (a BoxIndex over ``patches``) restricts both passes to the patches whose
    frame meets ``box``, in list order."""
    if index is not None:
        patches = index.query(box)
    shp = (box.ny, box.nx)
    out = Coarse(box, np.zeros((M,) + shp), np.zeros((M,) + shp), np.zeros((M,) + shp),
                 np.zeros(shp), np.zeros(shp, dtype=bool))

    def source(p, sj, si):
        if blend is None:
            return p.h[:, sj, si], p.hu[:, sj, si], p.hv[:, sj, si]
        theta, stash = blend
        oh, ohu, ohv = stash[id(p)]
        w0 = 1.0 - theta
        return (w0 * oh[:, sj, si] + theta * p.h[:, sj, si],
                w0 * ohu[:, sj, si] + theta * p.hu[:, sj, si],
                w0 * ohv[:, sj, si] + theta * p.hv[:, sj, si])

    for p in patches:
        reg = box.meet(p.box)
        if reg is None:
            continue
        sj, si = p.sl(reg)
        dj = slice(reg.lo_j - box.lo_j, reg.hi_j - box.lo_j + 1)
        di = slice(reg.lo_i - box.lo_i, reg.hi_i - box.lo_i + 1)
        h, hu, hv = source(p, sj, si)
        out.h[:, dj, di] = h
        out.hu[:, dj, di] = hu
        out.hv[:, dj, di] = hv
        out.bathy[dj, di] = p.bathy[sj, si]
        out.avail[dj, di] = True
    if include_ghosts:
        for p in patches:
            reg = box.meet(p.full)
            if reg is None:
                continue
            sj, si = p.sl(reg)
            dj = slice(reg.lo_j - box.lo_j, reg.hi_j - box.lo_j + 1)
            di = slice(reg.lo_i - box.lo_i, reg.hi_i - box.lo_i + 1)
            need = ~out.avail[dj, di]
            if not need.any():
                continue
            h, hu, hv = source(p, sj, si)
            for dst, src in ((out.h, h), (out.hu, hu), (out.hv, hv)):
                view = dst[:, dj, di]
                view[:, need] = src[:, need]
            bview = out.bathy[dj, di]
            bview[need] = p.bathy[sj, si][need]
            aview = out.avail[dj, di]
            aview[need] = True
    return out


def interpolate_state(c: Coarse, fbox: Box, fine_bathy: np.ndarray, rx: int, ry: int,
                      prm: Params):
    """refine.interpolate_state (refine.py:158-190) via the C restatement."""
    M = c.h.shape[0]
    ch = np.ascontiguousarray(c.h)
    chu = np.ascontiguousarray(c.hu)
    chv = np.ascontiguousarray(c.hv)
    cb = np.ascontiguousarray(c.bathy)
    ca = np.ascontiguousarray(c.avail, dtype=np.uint8)
    fb = np.ascontiguousarray(fine_bathy, dtype=np.float64)
    oh = np.zeros((M, fbox.ny, fbox.nx))
    ohu = np.zeros_like(oh)
    ohv = np.zeros_like(oh)
    st = lib().orc_interpolate_state(
        M, _p(ch), _p(chu), _p(chv), _p(cb), ca.ctypes.data_as(_u8p),
        c.box.lo_i, c.box.lo_j, c.box.nx, c.box.ny,
        fbox.lo_i, fbox.lo_j, fbox.nx, fbox.ny,
        _p(fb), fb.shape[1], rx, ry, prm.tol,
        _p(oh), _p(ohu), _p(ohv), fbox.nx, fbox.nx * fbox.ny)
    if st == 4:
        raise GeometryFault(f"fine box {fbox} has parents outside {c.box}")
    if st != 0:
        raise OracleError(f"orc_interpolate_state status {st}")
    return oh, ohu, ohv


def refine_patch(c: Coarse, fp: OPatch, rx: int, ry: int, prm: Params,
                 region: Optional[Box] = None, coarse_cell_area: Optional[float] = None):
    """refine.refine_patch (refine.py:193-239); returns fine - coarse mass."""
    region = fp.box if region is None else region
    if not fp.box.covers(region):
        raise GeometryFault(f"region {region} outside fine patch {fp.box}")
    foot = region.coarse(rx, ry)
    if not c.box.covers(foot):
        raise GeometryFault(f"{region} not inside coarse footprint {c.box}")
    fj = slice(foot.lo_j - c.box.lo_j, foot.hi_j - c.box.lo_j + 1)
    fi = slice(foot.lo_i - c.box.lo_i, foot.hi_i - c.box.lo_i + 1)
    if not c.avail[fj, fi].all():
        raise GeometryFault(f"coarse data under {region} incomplete")
    jj, ii = fp.sl(region)
    h, hu, hv = interpolate_state(c, region, fp.bathy[jj, ii], rx, ry, prm)
    fp.h[:, jj, ii] = h
    fp.hu[:, jj, ii] = hu
    fp.hv[:, jj, ii] = hv
    af = fp.spec.dx * fp.spec.dy
    if coarse_cell_area is None:
        coarse_cell_area = (fp.spec.dx * rx) * (fp.spec.dy * ry)
    return h.sum(axis=(1, 2)) * af - c.h[:, fj, fi].sum(axis=(1, 2)) * coarse_cell_area


def block_mean(a: np.ndarray, rx: int, ry: int) -> np.ndarray:
    """coarsen.block_mean (coarsen.py:21-27) in numpy's summation order."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    lead = a.shape[:-2]
    ny, nx = a.shape[-2:]
    if ny % ry or nx % rx:
        raise ValueError("shape not divisible by ratio")
    flat = a.reshape((-1, ny, nx))
    out = np.empty((flat.shape[0], ny // ry, nx // rx))
    for k in range(flat.shape[0]):
        lib().orc_block_mean(_p(flat[k]), nx, nx // rx, ny // ry, rx, ry, _p(out[k]), nx // rx)
    return out.reshape(lead + (ny // ry, nx // rx))


def average_down(fine, coarse, rx: int, ry: int, prm: Params, check_time: bool = True,
                 index: Optional[BoxIndex] = None):
    """coarsen.average_down (coarsen.py:30-76); ``index`` over ``coarse``."""
    if not fine or not coarse:
        return np.zeros(prm.M)
    if check_time:
        # every (fine, coarse) pair of the reference's double loop, over the
        # distinct clocks only (the same test, O(P) instead of O(P^2))
        ctimes = list(dict.fromkeys(cp.time for cp in coarse))
        for fp in fine:
            for ct in ctimes:
                if abs(fp.time - ct) > 1e-12 * max(1.0, abs(ct)):
                    raise TimeSyncFault(f"level {fp.level} t={fp.time!r} vs {ct!r}")
    delta = np.zeros(prm.M)
    for fp in fine:
        cb = fp.box.coarse(rx, ry)
        jj, ii = fp.inner
        avg = [block_mean(a[:, jj, ii], rx, ry) for a in (fp.h, fp.hu, fp.hv)]
        dry = avg[0] <= prm.tol
        avg[1][dry] = 0.0
        avg[2][dry] = 0.0
        for cp in (coarse if index is None else index.query(cb)):
            ov = cb.meet(cp.box)
            if ov is None:
                continue
            dj, di = cp.sl(ov)
            sj = slice(ov.lo_j - cb.lo_j, ov.hi_j - cb.lo_j + 1)
            si = slice(ov.lo_i - cb.lo_i, ov.hi_i - cb.lo_i + 1)
            delta += (avg[0][:, sj, si] - cp.h[:, dj, di]).sum(axis=(1, 2)) * (
                cp.spec.dx * cp.spec.dy)
            cp.h[:, dj, di] = avg[0][:, sj, si]
            cp.hu[:, dj, di] = avg[1][:, sj, si]
            cp.hv[:, dj, di] = avg[2][:, sj, si]
    return delta


# --------------------------------------------------------------------------
# boundary conditions and ghost filling (ghost.py:89-197)
# --------------------------------------------------------------------------
_SIDE_ORDER = ("left", "right", "bottom", "top")


def touching_sides(box: Box, level_box: Box):
    s = []
    if box.lo_i == level_box.lo_i:
        s.append("left")
    if box.hi_i == level_box.hi_i:
        s.append("right")
    if box.lo_j == level_box.lo_j:
        s.append("bottom")
    if box.hi_j == level_box.hi_j:
        s.append("top")
    return [x for x in _SIDE_ORDER if x in s]


def bc_side(a: np.ndarray, side: str, kind: str, sign: float) -> None:
    """Wall: mirror with parity ``sign``; outflow: copy the first interior
    row/column (ghost.py:89-106)."""
    g = GHOST
    for k in range(g):
        if side == "left":
            a[..., :, g - 1 - k] = sign * a[..., :, g + k] if kind == "wall" else a[..., :, g]
        elif side == "right":
            a[..., :, -g + k] = sign * a[..., :, -g - 1 - k] if kind == "wall" else a[..., :, -g - 1]
        elif side == "bottom":
            a[..., g - 1 - k, :] = sign * a[..., g + k, :] if kind == "wall" else a[..., g, :]
        else:
            a[..., -g + k, :] = sign * a[..., -g - 1 - k, :] if kind == "wall" else a[..., -g - 1, :]


def apply_bathymetry_bcs(p: OPatch, bcs: dict, level_box: Box) -> None:
    for side in touching_sides(p.box, level_box):
        bc_side(p.bathy, side, bcs[side], 1.0)


def apply_state_bcs(p: OPatch, bcs: dict, level_box: Box) -> None:
    for side in touching_sides(p.box, level_box):
        xs = side in ("left", "right")
        for m in range(p.h.shape[0]):
            bc_side(p.h[m], side, bcs[side], 1.0)
            bc_side(p.hu[m], side, bcs[side], -1.0 if xs else 1.0)
            bc_side(p.hv[m], side, bcs[side], 1.0 if xs else -1.0)


def ghost_bands(box: Box):
    g = GHOST
    return [Box(box.lo_i - g, box.lo_j - g, box.hi_i + g, box.lo_j - 1),
            Box(box.lo_i - g, box.hi_j + 1, box.hi_i + g, box.hi_j + g),
            Box(box.lo_i - g, box.lo_j, box.lo_i - 1, box.hi_j),
            Box(box.hi_i + 1, box.lo_j, box.hi_i + g, box.hi_j)]


def fill_ghosts(p: OPatch, siblings, provider, bcs: dict, level_box: Box,
                rx: int, ry: int, prm: Params) -> None:
    """ghost.fill_ghosts (ghost.py:156-197): coarse interpolation, then
    sibling copies, then physical boundary conditions."""
    if provider is not None:
        for band in ghost_bands(p.box):
            dom = band.meet(level_box)
            if dom is None:
                continue
            pbox = Box(dom.lo_i // rx, dom.lo_j // ry, dom.hi_i // rx, dom.hi_j // ry).grow(1)
            c = provider(pbox)
            jj, ii = p.sl(dom)
            h, hu, hv = interpolate_state(c, dom, p.bathy[jj, ii], rx, ry, prm)
            p.h[:, jj, ii] = h
            p.hu[:, jj, ii] = hu
            p.hv[:, jj, ii] = hv
    for s in siblings:
        if s is p:
            continue
        ov = p.full.meet(s.box)
        if ov is None:
            continue
        dj, di = p.sl(ov)
        sj, si = s.sl(ov)
        p.h[:, dj, di] = s.h[:, sj, si]
        p.hu[:, dj, di] = s.hu[:, sj, si]
        p.hv[:, dj, di] = s.hv[:, sj, si]
    apply_state_bcs(p, bcs, level_box)


# --------------------------------------------------------------------------
# morphology, flagging and clustering (mesh.py:116-141, regrid.py:58-232)
# --------------------------------------------------------------------------
def dilate(mask: np.ndarray, w: int) -> np.ndarray:
    out = mask.copy()
    for _ in range(w):
        pad = np.pad(out, 1, constant_values=False)
        nxt = np.zeros_like(out)
        for dj in range(3):
            for di in range(3):
                nxt |= pad[dj:dj + out.shape[0], di:di + out.shape[1]]
        out = nxt
    return out


def erode(mask: np.ndarray, w: int) -> np.ndarray:
    out = mask.copy()
    for _ in range(w):
        pad = np.pad(out, 1, constant_values=True)
        nxt = np.ones_like(out)
        for dj in range(3):
            for di in range(3):
                nxt &= pad[dj:dj + out.shape[0], di:di + out.shape[1]]
        out = nxt
    return out


def surfaces(h: np.ndarray, bathy: np.ndarray) -> np.ndarray:
    """state.surfaces_from_state (state.py:56-61)."""
    return np.cumsum(h[::-1], axis=0)[::-1] + bathy


def depths_from_surfaces(eta: np.ndarray, bathy: np.ndarray) -> np.ndarray:
    """state.state_from_surfaces (state.py:72-101), depths only."""
    M = eta.shape[0]
    h = np.zeros_like(eta)
    bhat = np.zeros_like(eta[0]) + bathy
    for m in range(M - 1, -1, -1):
        h[m] = np.maximum(eta[m] - bhat, 0.0)
        bhat = bhat + h[m]
    return h


def rest_surfaces(bathy: np.ndarray, eta_rest, prm: Params) -> np.ndarray:
    """scenario.rest_surfaces (scenario.py:81-96)."""
    eta = np.broadcast_to(np.asarray(eta_rest, float).reshape((-1,) + (1,) * bathy.ndim),
                          (len(eta_rest),) + bathy.shape)
    return surfaces(depths_from_surfaces(eta, bathy), bathy)


def flag_reference(patches, spec: Spec, prm: Params, eta_rest, wave_tol, buffer_w: int):
    """regrid.flag_cells (regrid.py:58-101)."""
    shp = (spec.ny, spec.nx)
    flags = np.zeros(shp, bool)
    covered = np.zeros(shp, bool)
    wet = np.zeros((prm.M,) + shp, bool)
    for p in patches:
        jj, ii = p.inner
        h = p.h[:, jj, ii]
        b = p.bathy[jj, ii]
        eta = surfaces(h, b)
        er = rest_surfaces(b, eta_rest, prm)
        dj = slice(p.box.lo_j, p.box.hi_j + 1)
        di = slice(p.box.lo_i, p.box.hi_i + 1)
        covered[dj, di] = True
        f = np.zeros(h.shape[1:], bool)
        for m in range(prm.M):
            f |= np.abs(eta[m] - er[m]) > wave_tol[m]
        flags[dj, di] = f
        wet[:, dj, di] = h > prm.tol
    for m in range(prm.M):
        # dry is "covered and not wet" (regrid.py:91-92)
        flags |= wet[m] & dilate(covered & ~wet[m], buffer_w)
    return dilate(flags, buffer_w) & covered


def nesting_allowed(patches, spec: Spec) -> np.ndarray:
    """regrid.nesting_allowed (regrid.py:185-211) without physical regions."""
    m = np.zeros((spec.ny, spec.nx), bool)
    for p in patches:
        m[p.box.lo_j:p.box.hi_j + 1, p.box.lo_i:p.box.hi_i + 1] = True
    return erode(m, 1)


def _best_cut(sig: np.ndarray):
    """regrid._signature_cut (regrid.py:104-126): (index, quality) or None."""
    n = sig.size
    if n < 2:
        return None
    zero = np.flatnonzero(sig == 0)
    if zero.size:
        brk = np.flatnonzero(np.diff(zero) != 1) + 1
        runs = [r for r in np.split(zero, brk) if r[0] > 0 and r[-1] < n - 1]
        if runs:
            longest = runs[0]
            for r in runs[1:]:
                if len(r) > len(longest):
                    longest = r
            return int(longest[len(longest) // 2]), 2
    if n >= 4:
        lap = sig[2:] - 2 * sig[1:-1] + sig[:-2]
        jump = np.abs(np.diff(lap))
        if jump.size and jump.max() > 0:
            return int(np.argmax(jump)) + 2, 1
    return n // 2, 0


def cluster_flags(flags: np.ndarray, eff: float, allowed: Optional[np.ndarray] = None):
    """regrid.cluster_flags (regrid.py:129-182): recursive bisection."""
    if allowed is not None and (flags & ~allowed).any():
        raise ValueError("flags outside the allowed region")
    boxes = []
    stack = [(0, 0, flags.shape[1] - 1, flags.shape[0] - 1)]
    while stack:
        i0, j0, i1, j1 = stack.pop()
        sub = flags[j0:j1 + 1, i0:i1 + 1]
        rows = np.flatnonzero(sub.any(axis=1))
        if rows.size == 0:
            continue
        cols = np.flatnonzero(sub.any(axis=0))
        a_j, b_j = j0 + int(rows[0]), j0 + int(rows[-1])
        a_i, b_i = i0 + int(cols[0]), i0 + int(cols[-1])
        sub = flags[a_j:b_j + 1, a_i:b_i + 1]
        area = sub.size
        ok = allowed is None or bool(allowed[a_j:b_j + 1, a_i:b_i + 1].all())
        if area == 1 or (ok and int(sub.sum()) >= eff * area):
            boxes.append(Box(a_i, a_j, b_i, b_j))
            continue
        cx = _best_cut(sub.sum(axis=0))
        cy = _best_cut(sub.sum(axis=1))
        if cx is None and cy is None:
            boxes.append(Box(a_i, a_j, b_i, b_j))
            continue
        sx = (-1, 0) if cx is None else (cx[1], b_i - a_i + 1)
        sy = (-1, 0) if cy is None else (cy[1], b_j - a_j + 1)
        # depth-first, first half first: push the second half below the first
        if sx >= sy:
            c = cx[0]
            stack.append((a_i + c, a_j, b_i, b_j))
            stack.append((a_i, a_j, a_i + c - 1, b_j))
        else:
            c = cy[0]
            stack.append((a_i, a_j + c, b_i, b_j))
            stack.append((a_i, a_j, b_i, a_j + c - 1))
    return sorted(boxes, key=lambda b: (b.lo_j, b.lo_i))


def chop_boxes(boxes, max_nx: int, max_ny: int, aligned: bool = False):
    """Harness max-patch-size chop: each box is cut into
    tiles of at most max_nx x max_ny coarse cells (from the box corner, or
    at global multiples of the tile size when ``aligned``), then the list is
    re-sorted like cluster_flags' output."""
    out = []
    for b in boxes:
        ys = []
        j = b.lo_j
        while j <= b.hi_j:
            nj = ((j // max_ny) + 1) * max_ny if aligned else j + max_ny
            ys.append((j, min(nj - 1, b.hi_j)))
            j = nj
        xs = []
        i = b.lo_i
        while i <= b.hi_i:
            ni = ((i // max_nx) + 1) * max_nx if aligned else i + max_nx
            xs.append((i, min(ni - 1, b.hi_i)))
            i = ni
        for (j0, j1) in ys:
            for (i0, i1) in xs:
                out.append(Box(i0, j0, i1, j1))
    return sorted(out, key=lambda b: (b.lo_j, b.lo_i))


def row_runs(mask: np.ndarray, box: Box):
    """regrid._row_runs (regrid.py:214-232)."""
    out = []
    for j in range(mask.shape[0]):
        idx = np.flatnonzero(mask[j])
        if idx.size == 0:
            continue
        brk = np.flatnonzero(np.diff(idx) != 1) + 1
        for run in np.split(idx, brk):
            out.append(Box(box.lo_i + int(run[0]), box.lo_j + j,
                           box.lo_i + int(run[-1]), box.lo_j + j))
    return out


# --------------------------------------------------------------------------
# regrid data movement (regrid.py:235-371)
# --------------------------------------------------------------------------
def _coverage(boxes, spec: Spec, rx: int, ry: int, coarse_given: bool = False):
    cov = np.zeros((spec.ny, spec.nx), bool)
    for b in boxes:
        cb = b if coarse_given else b.coarse(rx, ry)
        cov[cb.lo_j:cb.hi_j + 1, cb.lo_i:cb.hi_i + 1] = True
    return cov


def check_bathymetry_consistency(fp: OPatch, coarse, rx: int, ry: int, atol: float = 1e-12,
                                 index: Optional[BoxIndex] = None):
    """coarsen.check_bathymetry_consistency (coarsen.py:79-100)."""
    cb = fp.box.coarse(rx, ry)
    if index is not None:
        coarse = index.query(cb)
    jj, ii = fp.inner
    avg = block_mean(fp.bathy[jj, ii], rx, ry)
    for cp in coarse:
        ov = cb.meet(cp.box)
        if ov is None:
            continue
        dj, di = cp.sl(ov)
        sj = slice(ov.lo_j - cb.lo_j, ov.hi_j - cb.lo_j + 1)
        si = slice(ov.lo_i - cb.lo_i, ov.hi_i - cb.lo_i + 1)
        err = np.abs(avg[sj, si] - cp.bathy[dj, di]).max()
        if err > atol:
            raise AssertionError(f"bathymetry ladder does not telescope under {fp.box}: {err:.3e}")


# --------------------------------------------------------------------------
# the subcycled driver (driver.py:89-362) over a harness problem
# --------------------------------------------------------------------------
@dataclass
class Stats:
    total_cell_updates: int = 0
    cell_updates_per_level: dict = field(default_factory=dict)
    num_coarse_steps: int = 0
    num_regrids: int = 0
    hyperbolicity_warnings: int = 0
    wet_prefix_repairs: int = 0
    clipped_mass: list = field(default_factory=list)
    refine_delta: list = field(default_factory=list)
    derefine_delta: list = field(default_factory=list)
    sync_delta: list = field(default_factory=list)
    initial_mass: list = field(default_factory=list)


class Simulation:
    """Oracle of driver.Simulation (driver.py:89-362).

    ``problem`` is a harness problem (paper_1803_01450_b200.problems):
    geometry, parameters, seeded input fields and the harness plumbing of
    SURVEY.md App. B (flag rules, max-patch chop, dynamic r_t, fixed initial
    layouts).  The oracle implements those rules itself from the problem's
    parameters.
    """

    def __init__(self, problem, check_nesting: bool = False, workers: int = 1):
        self.pb = problem
        self.workers = max(1, int(workers))
        self._pool = None
        if self.workers > 1:
            from concurrent.futures import ThreadPoolExecutor
            self._pool = ThreadPoolExecutor(self.workers)
        self.prm = Params(problem.num_layers, tuple(problem.densities), problem.gravity,
                          problem.dry_tolerance)
        self.specs = [Spec(*s) for s in problem.level_specs()]
        self.L = len(self.specs)
        self.patches = {s.level: [] for s in self.specs}
        self.steps = {s.level: 0 for s in self.specs}
        self.stats = Stats()
        M = self.prm.M
        self.stats.clipped_mass = [0.0] * M
        self.stats.refine_delta = [0.0] * M
        self.stats.derefine_delta = [0.0] * M
        self.stats.sync_delta = [0.0] * M
        self._stash = {}
        self._event = np.zeros(M)
        self.time = 0.0
        base = self._new_patch(1, self.level_box(1))
        self._init_from_problem(base)
        self.patches[1].append(base)
        for lev in range(1, self.L):
            self._rebuild(lev, init=True)
        self._mass_prev = self.composite_mass()
        self.stats.initial_mass = list(self._mass_prev)

    # -- helpers ----------------------------------------------------------
    def spec(self, level: int) -> Spec:
        return self.specs[level - 1]

    def _index(self, level: int) -> BoxIndex:
        """BoxIndex over the level's current patch list (rebuilt when a
        regrid replaces the list)."""
        cache = self.__dict__.setdefault("_idx", {})
        ix = cache.get(level)
        pats = self.patches[level]
        if ix is None or ix.patches is not pats or ix.n != len(pats):
            ix = BoxIndex(pats)
            cache[level] = ix
        return ix

    def level_box(self, level: int) -> Box:
        s = self.spec(level)
        return Box(0, 0, s.nx - 1, s.ny - 1)

    def _new_patch(self, level: int, box: Box) -> OPatch:
        p = OPatch(self.spec(level), box, self.prm.M)
        p.bathy[:, :] = self.pb.bathymetry_box(level, p.full)
        apply_bathymetry_bcs(p, self.pb.boundaries, self.level_box(level))
        return p

    def _init_from_problem(self, p: OPatch) -> None:
        h, hu, hv = self.pb.initial_state_box(p.level, p.full)
        p.h[...] = h
        p.hu[...] = hu
        p.hv[...] = hv

    # -- mass accounting (driver.py:138-153) ------------------------------
    def composite_mass(self) -> np.ndarray:
        tot = np.zeros(self.prm.M)
        for lev in range(1, self.L + 1):
            s = self.spec(lev)
            if lev < self.L:
                cov = _coverage([p.box for p in self.patches[lev + 1]], s, s.r_x, s.r_y)
            else:
                cov = np.zeros((s.ny, s.nx), bool)
            for p in self.patches[lev]:
                jj, ii = p.inner
                w = ~cov[p.box.lo_j:p.box.hi_j + 1, p.box.lo_i:p.box.hi_i + 1]
                tot += (p.h[:, jj, ii] * w[None]).sum(axis=(1, 2)) * (s.dx * s.dy)
        return tot

    # -- ghost filling (driver.py:157-190) ---------------------------------
    def _provider(self, level: int, t: float):
        if level == 1:
            return None
        parents = self.patches[level - 1]
        blend = None
        st = self._stash.get(level - 1)
        if st is not None:
            t0, dt, old = st
            theta = min(1.0, max(0.0, (t - t0) / dt)) if dt > 0 else 1.0
            blend = (theta, old)
        M = self.prm.M
        index = self._index(level - 1)
        return lambda box: gather(parents, box, M, blend=blend, index=index)

    def fill_level_ghosts(self, level: int, t: float) -> None:
        ps = self.spec(level - 1) if level > 1 else None
        prov = self._provider(level, t)
        sib = self.patches[level]
        index = self._index(level)
        for p in sib:
            # the siblings whose interior can meet p's frame, in list order
            fill_ghosts(p, index.query(p.full), prov, self.pb.boundaries, self.level_box(level),
                        ps.r_x if ps else 1, ps.r_y if ps else 1, self.prm)

    # -- regridding (driver.py:192-222, regrid.py:235-353) ------------------
    def flags_for(self, level: int) -> np.ndarray:
        s = self.spec(level)
        rule = self.pb.flag_rule
        kind = rule[0]
        pats = self.patches[level]
        if kind == "reference":
            return flag_reference(pats, s, self.prm, self.pb.eta_rest,
                                  self.pb.wave_tolerance, self.pb.buffer_width)
        covered = np.zeros((s.ny, s.nx), bool)
        for p in pats:
            covered[p.box.lo_j:p.box.hi_j + 1, p.box.lo_i:p.box.hi_i + 1] = True
        if kind == "gradient":
            from paper_1803_01450_b200.problems import gradient_flags_map
            layers = rule[3]
            eta = np.zeros((len(layers), s.ny, s.nx))
            for p in pats:
                jj, ii = p.inner
                e = surfaces(p.h[:, jj, ii], p.bathy[jj, ii])
                eta[:, p.box.lo_j:p.box.hi_j + 1, p.box.lo_i:p.box.hi_i + 1] = e[list(layers)]
            f = gradient_flags_map(eta, covered, s.dx, s.dy, rule[1])
            return dilate(f, rule[2]) & covered
        if kind == "bernoulli":
            f = self.pb.bernoulli_flags(level, self.steps[level])
            return dilate(f, rule[2]) & covered
        raise ValueError(kind)

    def _rebuild(self, level: int, init: bool = False) -> bool:
        s = self.spec(level)
        rx, ry = s.r_x, s.r_y
        old = self.patches[level + 1]
        sync_time = self.patches[level][0].time if self.patches[level] else 0.0
        fixed = self.pb.fixed_layout(level + 1) if init else None
        if fixed is not None:
            cboxes = sorted([Box(*b).coarse(rx, ry) for b in fixed],
                            key=lambda b: (b.lo_j, b.lo_i))
        else:
            flags = self.flags_for(level)
            allowed = nesting_allowed(self.patches[level], s)
            flags &= allowed
            cboxes = cluster_flags(flags, self.pb.efficiency_target, allowed)
            if self.pb.max_patch is not None:
                cboxes = chop_boxes(cboxes, *self.pb.max_patch, aligned=self.pb.chop_aligned)
        nboxes = [b.fine(rx, ry) for b in cboxes]
        key = lambda b: (b.lo_j, b.lo_i)
        if sorted(nboxes, key=key) == sorted((p.box for p in old), key=key):
            return False
        old_cov = _coverage([p.box for p in old], s, rx, ry)
        old_index = BoxIndex(old)
        carea = s.dx * s.dy
        M = self.prm.M
        rdelta = np.zeros(M)
        new = []
        for fb, cb in zip(nboxes, cboxes):
            p = self._new_patch(level + 1, fb)
            p.time = sync_time
            check_bathymetry_consistency(p, self.patches[level], rx, ry, index=self._index(level))
            if init and fixed is None and self.pb.init_mode == "scenario":
                self._init_from_problem(p)
            else:
                mask = ~old_cov[cb.lo_j:cb.hi_j + 1, cb.lo_i:cb.hi_i + 1]
                for run in row_runs(mask, cb):
                    c = gather(self.patches[level], run.grow(1), M, include_ghosts=False,
                               index=self._index(level))
                    rdelta += refine_patch(c, p, rx, ry, self.prm, region=run.fine(rx, ry),
                                           coarse_cell_area=carea)
                for o in old_index.query(fb):
                    ov = fb.meet(o.box)
                    if ov is None:
                        continue
                    dj, di = p.sl(ov)
                    sj, si = o.sl(ov)
                    p.h[:, dj, di] = o.h[:, sj, si]
                    p.hu[:, dj, di] = o.hu[:, sj, si]
                    p.hv[:, dj, di] = o.hv[:, sj, si]
            new.append(p)
        new_cov = _coverage(cboxes, s, rx, ry, coarse_given=True)
        ddelta = np.zeros(M)
        gone = old_cov & ~new_cov
        if gone.any():
            fs = self.spec(level + 1)
            for o in old:
                cb = o.box.coarse(rx, ry)
                sub = gone[cb.lo_j:cb.hi_j + 1, cb.lo_i:cb.hi_i + 1]
                if not sub.any():
                    continue
                fmask = np.repeat(np.repeat(sub, ry, axis=0), rx, axis=1)
                jj, ii = o.inner
                fmass = (o.h[:, jj, ii] * fmask[None]).sum(axis=(1, 2)) * (fs.dx * fs.dy)
                cv = np.zeros(M)
                for cp in self._index(level).query(cb):
                    ov = cb.meet(cp.box)
                    if ov is None:
                        continue
                    dj, di = cp.sl(ov)
                    m2 = sub[ov.lo_j - cb.lo_j:ov.hi_j - cb.lo_j + 1,
                             ov.lo_i - cb.lo_i:ov.hi_i - cb.lo_i + 1]
                    cv += (cp.h[:, dj, di] * m2[None]).sum(axis=(1, 2))
                ddelta += cv * carea - fmass
        self.patches[level + 1] = new
        if not init:
            self.stats.num_regrids += 1
            for m in range(M):
                self.stats.refine_delta[m] += rdelta[m]
                self.stats.derefine_delta[m] += ddelta[m]
            self._event += rdelta + ddelta
        return True

    def regrid_from(self, level: int) -> None:
        if self._rebuild(level):
            for deeper in range(level + 1, self.L):
                self._rebuild(deeper)

    # -- stepping (driver.py:224-309) ----------------------------------------
    def _step_patches(self, level: int, dt: float) -> None:
        y_first = bool(self.steps[level] % 2)
        n = 0
        pats = self.patches[level]
        # the C step releases the GIL (ctypes), so worker threads run patches
        # concurrently, like the reference's ThreadPoolExecutor (driver.py:231)
        if self._pool is not None and len(pats) > 1:
            results = list(self._pool.map(lambda p: step_patch(p, dt, self.prm, y_first=y_first), pats))
        else:
            results = [step_patch(p, dt, self.prm, y_first=y_first) for p in pats]
        for r in results:
            n += r.cells_updated
            self.stats.hyperbolicity_warnings += r.hyperbolicity_fixes
            self.stats.wet_prefix_repairs += r.wet_prefix_repairs
            for m in range(self.prm.M):
                self.stats.clipped_mass[m] += float(r.clipped_mass[m])
        self.stats.total_cell_updates += n
        self.stats.cell_updates_per_level[level] = self.stats.cell_updates_per_level.get(level, 0) + n

    def advance_level(self, level: int, dt: float, t0: float) -> None:
        if level < self.L and self.steps[level] % self.pb.regrid_interval == 0:
            self.regrid_from(level)
        self.fill_level_ghosts(level, t0)
        pats = self.patches[level]
        child = self.patches.get(level + 1)
        old = None
        if child:
            old = {id(p): (p.h.copy(), p.hu.copy(), p.hv.copy()) for p in pats}
        self._step_patches(level, dt)
        self.steps[level] += 1
        t1 = t0 + dt
        for p in pats:
            p.time = t1
        if child:
            self.fill_level_ghosts(level, t1)
            self._stash[level] = (t0, dt, old)
            s = self.spec(level)
            dtf = dt / s.r_t
            for k in range(s.r_t):
                self.advance_level(level + 1, dtf, t0 + k * dtf)
            for p in self.patches[level + 1]:
                p.time = t1
            average_down(self.patches[level + 1], pats, s.r_x, s.r_y, self.prm, index=self._index(level))
            del self._stash[level]

    def check_finite(self) -> None:
        for lev, pats in self.patches.items():
            for p in pats:
                if not (np.isfinite(p.h).all() and np.isfinite(p.hu).all()
                        and np.isfinite(p.hv).all()):
                    raise NumericalAbort(f"non-finite state on level {lev} patch {p.box}")

    def level_speed(self, level: int) -> float:
        sp = 0.0
        for p in self.patches[level]:
            sp = max(sp, observed_max_speed(p, self.prm))
        return sp

    def choose_dt(self) -> float:
        dt = self.pb.dt_max
        for p in self.patches[1]:
            dt = min(dt, stable_dt(p, self.prm, self.pb.cfl, self.pb.dt_max))
        return dt

    def apply_dynamic_rt(self, dt: float) -> None:
        """Harness dynamic r_t: per coarse step, the
        smallest r_t <= max(r_x, r_y) keeping the finer level's observed
        Courant number <= cfl."""
        if not self.pb.dynamic_rt:
            return
        dtl = dt
        for lev in range(1, self.L):
            s = self.spec(lev)
            fs = self.spec(lev + 1)
            sp = self.level_speed(lev + 1)
            rmax = max(s.r_x, s.r_y)
            rt = self.pb.pick_rt(sp, dtl, min(fs.dx, fs.dy), rmax)
            self.specs[lev - 1] = replace(s, r_t=rt)
            dtl = dtl / rt

    def advance_coarse_step(self, dt: float) -> None:
        self._event[:] = 0.0
        self.advance_level(1, dt, self.time)
        self.time += dt
        mass = self.composite_mass()
        sync = mass - self._mass_prev - self._event
        for m in range(self.prm.M):
            self.stats.sync_delta[m] += float(sync[m])
        self._mass_prev = mass
        self.stats.num_coarse_steps += 1
        self.check_finite()

    def run(self, n_coarse: int):
        for _ in range(n_coarse):
            dt = self.choose_dt()
            self.apply_dynamic_rt(dt)
            self.advance_coarse_step(dt)
        return self.stats
