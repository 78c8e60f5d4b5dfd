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
                                    pool.n_tiles, _params(params), pool.speed_bits.data_ptr(),
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
    N.check(L.mlamr_step(lv, src.data_ptr(), dst.data_ptr(), pool.tiles_d.data_ptr(), pool.n_tiles, dt,
                         int(bool(y_first)), prm, pool.speed_bits.data_ptr(), pool.tile_acc.data_ptr(),
                         status.data_ptr(), sh), "step")
    N.check(L.mlamr_step_finalize(lv, src.data_ptr(), dst.data_ptr(), pool.tiles_d.data_ptr(), pool.n_tiles,
                                  dt, prm, pool.speed_bits.data_ptr(), pool.tile_acc.data_ptr(),
                                  acc.data_ptr(), status.data_ptr(), bad.data_ptr(), sh), "finalize")
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
