"""Drop-in shims with the reference's per-patch signatures.

Each function accepts the reference's objects (anything shaped like
``mlamr.mesh.Patch``: ``h, hu, hv`` [M, ny+4, nx+4] and ``bathy`` numpy
arrays, ``box``, ``dx``/``dy`` or ``spec``, ``ghost_width`` = 2) and runs
the computation on the GPU through ``libmlamr_b200.so`` as a batch of
one, mutating the arrays in place exactly like the reference:

* :func:`step_patch`        physics.step_patch        (physics.py:330-386)
* :func:`stable_dt`         physics.stable_dt         (physics.py:281-289)
* :func:`interpolate_state` refine.interpolate_state  (refine.py:158-190)
* :func:`refine_patch`      refine.refine_patch       (refine.py:193-239)
* :func:`average_down`      coarsen.average_down      (coarsen.py:30-76)
* :func:`check_bathymetry_consistency`  coarsen.check_bathymetry_consistency (coarsen.py:79-100)
* :func:`fill_ghosts`       ghost.fill_ghosts         (ghost.py:156-197)

They exist for integration and per-operation parity; the level-batched
:class:`~paper_1803_01450_b200.driver.Simulation` is the performance path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .device import LevelPool, empty_level_struct
from .errors import CflViolationError, GeometryError, TimeSyncError, raise_status
from .mesh import GHOST_WIDTH, IndexBox, LevelSpec


@dataclass
class StepResult:
    """physics.StepResult (physics.py:42-51)."""
    max_wave_speed: float
    cells_updated: int
    mass_delta: np.ndarray
    hyperbolicity_fixes: int = 0
    wet_prefix_repairs: int = 0
    clipped_mass: np.ndarray = field(default_factory=lambda: np.zeros(0))


def _params(params) -> N.Params:
    dens = tuple(params.densities)
    return N.make_params(params.num_layers, dens, params.gravity, params.dry_tolerance)


def _box(patch) -> IndexBox:
    b = patch.box
    return IndexBox(int(b[0]), int(b[1]), int(b[2]), int(b[3]))


def _dxdy(patch):
    if hasattr(patch, "dx"):
        return float(patch.dx), float(patch.dy)
    return float(patch.spec.dx), float(patch.spec.dy)


def _pool_for(patches, level_nx, level_ny, dx, dy, M, need_gown=False):
    spec = LevelSpec(1, level_nx, level_ny, dx, dy)
    dev = torch.device("cuda")
    stream = torch.cuda.current_stream(dev)
    boxes = np.asarray([tuple(_box(p)) for p in patches], dtype=np.int64)
    pool = LevelPool(spec, boxes, M, dev, stream, need_gown=need_gown)
    pool.upload_patches([(p.h, p.hu, p.hv) for p in patches])
    pool.upload_patches([p.bathy for p in patches], bathy=True)
    return pool


def _download_into(pool: LevelPool, patches, state=None, interior_only=False):
    host = pool.download(state)
    g = GHOST_WIDTH
    for k, p in enumerate(patches):
        h, hu, hv, _ = pool.patch_arrays(k, host=host)
        if interior_only:
            p.h[:, g:-g, g:-g] = h[:, g:-g, g:-g]
            p.hu[:, g:-g, g:-g] = hu[:, g:-g, g:-g]
            p.hv[:, g:-g, g:-g] = hv[:, g:-g, g:-g]
        else:
            p.h[...] = h
            p.hu[...] = hu
            p.hv[...] = hv


def observed_max_speed(patch, params) -> float:
    M = params.num_layers
    dx, dy = _dxdy(patch)
    b = _box(patch)
    pool = _pool_for([patch], b.hi_i + 1, b.hi_j + 1, dx, dy, M)
    L = N.lib()
    N.check(L.mlamr_max_speed_tiles(pool.struct(), pool.state.data_ptr(), pool.tiles_d.data_ptr(),
                                    pool.n_tiles, pool.tile_tx, _params(params), pool.speed_bits.data_ptr(),
                                    torch.cuda.current_stream().cuda_stream), "max_speed")
    bits = int(pool.speed_bits[0].item())
    return 0.0 if bits < 0 else float(np.array([bits], np.int64).view(np.float64)[0])


def stable_dt(patch, params, cfl_target: float, dt_max: float = 1.0) -> float:
    speed = observed_max_speed(patch, params)
    if speed <= 0.0:
        return dt_max
    dx, dy = _dxdy(patch)
    return min(dt_max, cfl_target * min(dx, dy) / speed)


def step_patch(patch, dt: float, params, y_first: bool = False) -> StepResult:
    """physics.step_patch on the GPU (batch of one)."""
    M = params.num_layers
    dx, dy = _dxdy(patch)
    b = _box(patch)
    pool = _pool_for([patch], b.hi_i + 1, b.hi_j + 1, dx, dy, M)
    L = N.lib()
    sh = torch.cuda.current_stream().cuda_stream
    prm = _params(params)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    bad = torch.full((1,), 2 ** 31 - 1, dtype=torch.int32, device="cuda")
    acc = torch.zeros(M + 2, dtype=torch.float64, device="cuda")
    src, dst = pool.state, pool.other
    dst.copy_(src)  # ghost frame of the result = input frame
    lv = pool.struct(src)
    N.check(L.mlamr_step(lv, src.data_ptr(), dst.data_ptr(), pool.tiles_d.data_ptr(), pool.n_tiles, pool.tile_tx, dt,
                         int(bool(y_first)), prm, pool.speed_bits.data_ptr(), pool.tile_acc.data_ptr(),
                         status.data_ptr(), None, None, sh), "step")
    N.check(L.mlamr_step_finalize(lv, src.data_ptr(), dst.data_ptr(), pool.tiles_d.data_ptr(), pool.n_tiles,
                                  dt, prm, pool.speed_bits.data_ptr(), pool.tile_acc.data_ptr(),
                                  acc.data_ptr(), status.data_ptr(), bad.data_ptr(), 0, sh), "finalize")
    st = int(status.item())
    bits = int(pool.speed_bits[0].item())
    speed = 0.0 if bits < 0 else float(np.array([bits], np.int64).view(np.float64)[0])
    if st & N.ST_CFL:
        raise CflViolationError(
            f"Courant number {speed * dt / min(dx, dy):.3f} > 1 on level {getattr(patch, 'level', 1)} "
            f"patch {tuple(b)}")
    raise_status(st)
    g = GHOST_WIDTH
    area = dx * dy
    # interior masses from the device (diagnostic, pairwise order differs)
    mb = np.array([patch.h[m, g:-g, g:-g].sum() for m in range(M)]) * area
    _download_into(pool, [patch], state=dst, interior_only=True)
    ma = np.array([patch.h[m, g:-g, g:-g].sum() for m in range(M)]) * area
    a = acc.cpu().numpy()
    return StepResult(max_wave_speed=speed, cells_updated=b.ncells, mass_delta=ma - mb,
                      hyperbolicity_fixes=int(round(a[M])), wet_prefix_repairs=int(round(a[M + 1])),
                      clipped_mass=a[:M].copy())


def interpolate_state(coarse, fine_box, fine_bathy, r_x: int, r_y: int, params):
    """refine.interpolate_state on the GPU: ``coarse`` is a CoarseData-like
    object (box, h, hu, hv, bathy, avail)."""
    M = params.num_layers
    cb = coarse.box
    fb = IndexBox(*[int(v) for v in fine_box])
    dev = "cuda"
    t = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dtype=dt)
    ch, chu, chv, cbat = t(coarse.h), t(coarse.hu), t(coarse.hv), t(coarse.bathy)
    cav = torch.from_numpy(np.ascontiguousarray(coarse.avail, dtype=np.uint8)).to(dev)
    fbt = t(fine_bathy)
    oh = torch.empty((M, fb.ny, fb.nx), dtype=torch.float64, device=dev)
    ohu = torch.empty_like(oh)
    ohv = torch.empty_like(oh)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    N.check(N.lib().mlamr_interpolate_box(M, ch.data_ptr(), chu.data_ptr(), chv.data_ptr(), cbat.data_ptr(),
                                          cav.data_ptr(), int(cb[0]), int(cb[1]), int(cb[2]) - int(cb[0]) + 1,
                                          int(cb[3]) - int(cb[1]) + 1, fb.lo_i, fb.lo_j, fb.nx, fb.ny,
                                          fbt.data_ptr(), r_x, r_y, _params(params), oh.data_ptr(),
                                          ohu.data_ptr(), ohv.data_ptr(), status.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream), "interpolate")
    if int(status.item()) & N.ST_GEOMETRY:
        raise GeometryError(f"fine box {tuple(fb)} has parents outside coarse data footprint {tuple(cb)}")
    return oh.cpu().numpy(), ohu.cpu().numpy(), ohv.cpu().numpy()


@dataclass
class CoarseData:
    """refine.CoarseData (refine.py:50-65): gathered coarse fields over a box."""
    box: tuple
    h: np.ndarray
    hu: np.ndarray
    hv: np.ndarray
    bathy: np.ndarray
    avail: np.ndarray

    @property
    def num_layers(self) -> int:
        return self.h.shape[0]


def _full_box(p) -> IndexBox:
    return _box(p).grown(GHOST_WIDTH)


def _local(p, b: IndexBox):
    fb = _full_box(p)
    j0, i0 = b.lo_j - fb.lo_j, b.lo_i - fb.lo_i
    return slice(j0, j0 + b.ny), slice(i0, i0 + b.nx)


def gather(patches, box, num_layers: int, blend=None, include_ghosts: bool = True) -> CoarseData:
    """ghost.gather (ghost.py:29-86): interiors first, then ghost frames as a
    fallback with the first patch in list order winning; optional time blend
    (1-theta)*old + theta*new with the stash keyed by id(patch).  Pure data
    assembly on the host (the numerical work happens in the kernels)."""
    b = IndexBox(*[int(v) for v in box])
    shp = (b.ny, b.nx)
    out = CoarseData(tuple(b), np.zeros((num_layers,) + shp), np.zeros((num_layers,) + shp),
                     np.zeros((num_layers,) + shp), np.zeros(shp), np.zeros(shp, dtype=bool))

    def src(p, sj, si):
        if blend is None:
            return p.h[:, sj, si], p.hu[:, sj, si], p.hv[:, sj, si]
        theta, stash = blend
        oh, ohu, ohv = stash[id(p)]
        w0 = 1.0 - theta
        return (w0 * oh[:, sj, si] + theta * p.h[:, sj, si], w0 * ohu[:, sj, si] + theta * p.hu[:, sj, si],
                w0 * ohv[:, sj, si] + theta * p.hv[:, sj, si])

    for interior in ((True, False) if include_ghosts else (True,)):
        for p in patches:
            reg = b.intersection(_box(p) if interior else _full_box(p))
            if reg is None:
                continue
            sj, si = _local(p, reg)
            dj = slice(reg.lo_j - b.lo_j, reg.hi_j - b.lo_j + 1)
            di = slice(reg.lo_i - b.lo_i, reg.hi_i - b.lo_i + 1)
            h, hu, hv = src(p, sj, si)
            if interior:
                out.h[:, dj, di], out.hu[:, dj, di], out.hv[:, dj, di] = h, hu, hv
                out.bathy[dj, di] = p.bathy[sj, si]
                out.avail[dj, di] = True
            else:
                need = ~out.avail[dj, di]
                if need.any():
                    for dst, v in ((out.h, h), (out.hu, hu), (out.hv, hv)):
                        view = dst[:, dj, di]
                        view[:, need] = v[:, need]
                    out.bathy[dj, di][need] = p.bathy[sj, si][need]
                    out.avail[dj, di][need] = True
    return out


def refine_patch(coarse, fine_patch, r_x: int, r_y: int, params, region=None, coarse_cell_area=None):
    """refine.refine_patch (refine.py:193-239) with the interpolation on the
    GPU; returns the per-layer mass delta fine - coarse."""
    pb = _box(fine_patch)
    region = pb if region is None else IndexBox(*[int(v) for v in region])
    if not pb.contains_box(region):
        raise GeometryError(f"region {tuple(region)} outside fine patch {tuple(pb)}")
    try:
        foot = region.coarsened(r_x, r_y)
    except ValueError as exc:
        raise GeometryError(str(exc)) from None
    cb = IndexBox(*[int(v) for v in coarse.box])
    if not cb.contains_box(foot):
        raise GeometryError(f"fine box {tuple(region)} not inside coarse data footprint {tuple(cb)}")
    fj = slice(foot.lo_j - cb.lo_j, foot.hi_j - cb.lo_j + 1)
    fi = slice(foot.lo_i - cb.lo_i, foot.hi_i - cb.lo_i + 1)
    if not np.asarray(coarse.avail)[fj, fi].all():
        raise GeometryError(f"coarse data under fine box {tuple(region)} is incomplete")
    jj, ii = _local(fine_patch, region)
    h, hu, hv = interpolate_state(coarse, tuple(region), fine_patch.bathy[jj, ii], r_x, r_y, params)
    fine_patch.h[:, jj, ii] = h
    fine_patch.hu[:, jj, ii] = hu
    fine_patch.hv[:, jj, ii] = hv
    dx, dy = _dxdy(fine_patch)
    if coarse_cell_area is None:
        coarse_cell_area = (dx * r_x) * (dy * r_y)
    return h.sum(axis=(1, 2)) * (dx * dy) - np.asarray(coarse.h)[:, fj, fi].sum(axis=(1, 2)) * coarse_cell_area


def average_down(fine_patches, coarse_patches, r_x: int, r_y: int, params, check_time: bool = True):
    """coarsen.average_down (coarsen.py:30-76): block means of every fine
    patch over the coarse interiors they cover (kernel K4), in place."""
    M = params.num_layers
    if not fine_patches or not coarse_patches:
        return np.zeros(M)
    if check_time:
        for fp in fine_patches:
            for cp in coarse_patches:
                if abs(fp.time - cp.time) > 1e-12 * max(1.0, abs(cp.time)):
                    raise TimeSyncError(f"level {getattr(fp, 'level', '?')} at t={fp.time!r} vs "
                                        f"level {getattr(cp, 'level', '?')} at t={cp.time!r}")
    cb = [_box(p) for p in coarse_patches]
    fbx = [_box(p) for p in fine_patches]
    cnx = max(b.hi_i for b in cb) + 1
    cny = max(b.hi_j for b in cb) + 1
    dxc, dyc = _dxdy(coarse_patches[0])
    dxf, dyf = _dxdy(fine_patches[0])
    coarse = _pool_for(coarse_patches, cnx, cny, dxc, dyc, M)
    fine = _pool_for(fine_patches, max(b.hi_i for b in fbx) + 1, max(b.hi_j for b in fbx) + 1, dxf, dyf, M)
    g = GHOST_WIDTH
    before = [p.h[:, g:-g, g:-g].copy() for p in coarse_patches]
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    bpp = fine.blocks_per_patch(fine.max_interior // (r_x * r_y))
    part = torch.zeros(fine.P * bpp * M, dtype=torch.float64, device="cuda")
    N.check(N.lib().mlamr_average_down(fine.struct(), coarse.struct(), r_x, r_y, _params(params),
                                       part.data_ptr(), bpp, status.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream), "average_down")
    _download_into(coarse, coarse_patches, interior_only=True)
    delta = np.zeros(M)
    for p, b0 in zip(coarse_patches, before):
        delta += (p.h[:, g:-g, g:-g] - b0).sum(axis=(1, 2)) * (dxc * dyc)
    return delta


def check_bathymetry_consistency(fine_patch, coarse_patches, r_x: int, r_y: int, atol: float = 1e-12) -> None:
    """coarsen.check_bathymetry_consistency (coarsen.py:79-100) on the GPU
    (mlamr_check_bathymetry): AssertionError when a covered coarse
    bathymetry value is not the block mean of its fine values."""
    if not coarse_patches:
        return
    fb = _box(fine_patch)
    cb = [_box(p) for p in coarse_patches]
    dxc, dyc = _dxdy(coarse_patches[0])
    dxf, dyf = _dxdy(fine_patch)
    coarse = _pool_for(coarse_patches, max(b.hi_i for b in cb) + 1, max(b.hi_j for b in cb) + 1, dxc, dyc, 1)
    fine = _pool_for([fine_patch], fb.hi_i + 1, fb.hi_j + 1, dxf, dyf, 1)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    bad = torch.full((1,), 2 ** 31 - 1, dtype=torch.int32, device="cuda")
    cbase, n = fine.coarse_base(r_x, r_y)
    N.check(N.lib().mlamr_check_bathymetry(fine.struct(), coarse.struct(), r_x, r_y, float(atol), cbase.data_ptr(),
                                           n, status.data_ptr(), bad.data_ptr(),
                                           torch.cuda.current_stream().cuda_stream), "check_bathymetry")
    if int(status.item()) & N.ST_BATHY:
        raise AssertionError(f"bathymetry ladder does not telescope under {tuple(fb)}")


def fill_ghosts(patch, siblings, parent_provider, boundaries, level_box, r_x: int, r_y: int, params) -> None:
    """ghost.fill_ghosts (ghost.py:156-197): coarse interpolation of every
    in-domain ghost band from ``parent_provider`` (GPU interpolation), then
    sibling copies and physical boundary conditions (kernel K2)."""
    M = params.num_layers
    pb = _box(patch)
    lb = IndexBox(*[int(v) for v in level_box])
    g = GHOST_WIDTH
    if parent_provider is not None:
        bands = [IndexBox(pb.lo_i - g, pb.lo_j - g, pb.hi_i + g, pb.lo_j - 1),
                 IndexBox(pb.lo_i - g, pb.hi_j + 1, pb.hi_i + g, pb.hi_j + g),
                 IndexBox(pb.lo_i - g, pb.lo_j, pb.lo_i - 1, pb.hi_j),
                 IndexBox(pb.hi_i + 1, pb.lo_j, pb.hi_i + g, pb.hi_j)]
        for band in bands:
            dom = band.intersection(lb)
            if dom is None:
                continue
            pbox = IndexBox(dom.lo_i // r_x, dom.lo_j // r_y, dom.hi_i // r_x, dom.hi_j // r_y).grown(1)
            c = parent_provider(pbox)
            jj, ii = _local(patch, dom)
            h, hu, hv = interpolate_state(c, tuple(dom), patch.bathy[jj, ii], r_x, r_y, params)
            patch.h[:, jj, ii] = h
            patch.hu[:, jj, ii] = hu
            patch.hv[:, jj, ii] = hv
    group = [patch] + [s for s in siblings if s is not patch]
    dx, dy = _dxdy(patch)
    pool = _pool_for(group, lb.hi_i + 1, lb.hi_j + 1, dx, dy, M)
    lv = pool.struct()
    lv.num_patches = 1  # fill only `patch`; the others serve as siblings
    N.check(N.lib().mlamr_fill_ghosts(lv, None, None, 0.0, 1, 1, N.bc_array(boundaries), _params(params),
                                      None, None, 0, torch.cuda.current_stream().cuda_stream), "fill_ghosts")
    host = pool.download()
    h, hu, hv, _ = pool.patch_arrays(0, host=host)
    patch.h[...] = h
    patch.hu[...] = hu
    patch.hv[...] = hv
