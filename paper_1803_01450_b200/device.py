"""Device-resident patch table and level pools.

One :class:`LevelPool` per level holds, in HBM:

* the patch table: int32 boxes [P, 4] and int64 element offsets [P];
* two state buffers (double buffering for the out-of-place step; the
  buffer a step read from is the driver's time-interpolation stash), each
  3M planes of ``field_stride`` float64 -- h_0..h_{M-1}, hu_*, hv_* -- with
  every patch a (ny+4) x (nx+4) row-major block (mesh.py:181-186) starting
  at a 256-byte aligned offset;
* one bathymetry plane of the same shape;
* int32 owner maps over the level's index space (+2-cell frame): interior
  owner (last in list order wins) and, for levels that act as parents,
  frame owner (first in list order wins) -- the gather precedence of
  ghost.py:29-86;
* the step work list: 16x32 interior tiles (patch, j0, i0).

PyTorch is used only as the allocator and stream provider; every kernel
is in ``libmlamr_b200.so`` (no CPU fallback).
"""

from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np
import torch

from . import _native as N
from .mesh import GHOST_WIDTH, LevelSpec

ALIGN = 32          # elements: patch blocks start on 256-byte boundaries
NTHREADS = 256


def _stream_handle(stream: torch.cuda.Stream) -> int:
    return stream.cuda_stream


class PinnedArena:
    """Pinned staging memory for small host->device uploads (patch tables,
    tile lists).  Copies from pageable memory would synchronise the stream
    (the driver stages them synchronously); staging through pinned memory
    keeps uploads asynchronous.  Regions are recycled after :meth:`reset`,
    which the driver calls at points where the stream has been drained."""

    def __init__(self, nbytes: int = 1 << 24):
        self.buf = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        self.off = 0
        self.spill = []   # oversize staging tensors kept alive until reset

    def reset(self) -> None:
        self.off = 0
        self.spill.clear()

    def upload(self, arr: np.ndarray, device, stream) -> torch.Tensor:
        a = np.ascontiguousarray(arr)
        n = a.nbytes
        dt = torch.from_numpy(a[:0]).dtype if a.size == 0 else torch.from_numpy(a.reshape(-1)[:1]).dtype
        if n == 0:
            return torch.empty(a.shape, dtype=dt, device=device)
        start = (self.off + 255) // 256 * 256
        if start + n <= self.buf.numel():
            host = self.buf[start:start + n]
            self.off = start + n
        else:
            host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
            self.spill.append(host)
        host.numpy()[:] = a.reshape(-1).view(np.uint8)
        with torch.cuda.stream(stream):
            out = torch.empty(a.shape, dtype=dt, device=device)
            out.view(-1).view(torch.uint8).copy_(host, non_blocking=True)
        return out


_ARENA = None

# Recycled device buffers: a regrid replaces a level's pool with one of
# similar size, so the retired state/bathymetry buffers are handed to the
# next pool instead of round-tripping GBs through cudaMalloc.  Reuse is
# stream-ordered (everything runs on the driver's stream).
_RECYCLE: list = []
ALLOC_STATS = {"fresh": 0, "fresh_bytes": 0, "reused": 0}
POOL_PROF = __import__("collections").defaultdict(float)   # host seconds inside LevelPool()


def dmemset(t: torch.Tensor, byte: int, stream) -> torch.Tensor:
    """Fill a contiguous device tensor with one byte value on ``stream``
    (cudaMemsetAsync, not a kernel): 0 for zero planes, 0xff for -1."""
    n = t.numel() * t.element_size()
    if n:
        rc = N.lib().mlamr_memset(t.data_ptr(), int(byte), n, _stream_handle(stream))
        if rc:
            raise N.NativeLibraryError(f"memset failed (cuda error {rc})")
    return t


def dzeros(n: int, dtype, device, stream) -> torch.Tensor:
    with torch.cuda.stream(stream):
        t = torch.empty(n, dtype=dtype, device=device)
    return dmemset(t, 0, stream)


def acquire(numel: int, dtype, device, stream) -> torch.Tensor:
    device = torch.device(device)
    if device.type == "cuda" and device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    best = None
    for k, t in enumerate(_RECYCLE):
        if t.dtype == dtype and t.device == device and t.numel() >= numel:
            if best is None or t.numel() < _RECYCLE[best].numel():
                best = k
    if best is not None and _RECYCLE[best].numel() <= 3 * numel + (1 << 20):
        t = _RECYCLE.pop(best)
        ALLOC_STATS["reused"] += 1
        return t[:numel]
    cap = int(numel * 1.5) + (1 << 16)
    ALLOC_STATS["fresh"] += 1
    ALLOC_STATS["fresh_bytes"] += cap * torch.tensor([], dtype=dtype).element_size()
    with torch.cuda.stream(stream):
        t = torch.empty(cap, dtype=dtype, device=device)
    return t[:numel]


def release(t: torch.Tensor) -> None:
    base = t._base if t._base is not None else t
    _RECYCLE.append(base)
    # bound the cache: keep the 16 largest buffers
    _RECYCLE.sort(key=lambda x: -x.numel())
    del _RECYCLE[16:]


# Recycled pinned host buffers for snapshots: cudaHostAlloc costs ~0.5 s per
# GB, so a snapshot taken inside a timed loop must not allocate.  Buffers
# are allocated with 50 % slack and handed back by Simulation.release_snapshot.
_PINNED: list = []


def pinned_acquire(numel: int, dtype) -> torch.Tensor:
    best = None
    for k, t in enumerate(_PINNED):
        if t.dtype == dtype and numel <= t.numel() <= 3 * numel + (1 << 20):
            if best is None or t.numel() < _PINNED[best].numel():
                best = k
    if best is not None:
        return _PINNED.pop(best)[:numel]
    return torch.empty(int(numel * 1.5) + (1 << 16), dtype=dtype, pin_memory=True)[:numel]


def pinned_release(t: torch.Tensor) -> None:
    base = t._base if t._base is not None else t
    _PINNED.append(base)
    _PINNED.sort(key=lambda x: -x.numel())
    del _PINNED[8:]


def reserve(nbytes: int, device, stream) -> None:
    """Warm the caching allocator with ``nbytes`` of device memory.

    Regrids replace level pools with ones of similar size; whenever a pool
    outgrows the recycled buffers its buffers come from cudaMalloc, which
    on a fresh GPU costs tens of milliseconds per GB (first-touch page
    mapping) inside the time loop.  One large allocation released into
    PyTorch's cache up front turns those into cache hits (cached blocks are
    split on demand)."""
    if nbytes <= 0:
        return
    free, _total = torch.cuda.mem_get_info(device)
    n = int(min(nbytes, 0.8 * free))
    if n <= 0:
        return
    with torch.cuda.stream(stream):
        t = torch.empty(n, dtype=torch.uint8, device=device)
        # allocations <= 1 MB come from the allocator's separate small pool
        # (2 MB segments): warm it too, or patch tables and partial-sum
        # buffers of a new pool occasionally reach cudaMalloc, which waits
        # for the queued steps and stalls the regrid by ~100 ms
        small = [torch.empty(1 << 19, dtype=torch.uint8, device=device) for _ in range(256)]
    del t, small


def arena() -> PinnedArena:
    global _ARENA
    if _ARENA is None:
        _ARENA = PinnedArena()
    return _ARENA


def tile_list(boxes: np.ndarray, shape: Optional[tuple] = None) -> np.ndarray:
    """(patch, j0, i0) for every step tile, patch-major; ``shape`` = (rows,
    columns), by default the library's choice for these boxes."""
    if len(boxes) == 0:
        return np.zeros((0, 3), np.int32)
    if shape is None:
        shape = N.step_tile(int((boxes[:, 2] - boxes[:, 0] + 1).max()), 2)
    TILE_Y, TILE_X = shape
    b = np.ascontiguousarray(boxes, dtype=np.int64).reshape(-1, 4)
    L = N.lib()
    n = int(L.mlamr_tile_list(b.ctypes.data, len(b), int(TILE_Y), int(TILE_X), None))
    out = np.empty((n, 3), np.int32)
    L.mlamr_tile_list(b.ctypes.data, len(b), int(TILE_Y), int(TILE_X), out.ctypes.data)
    return out


class LevelPool:
    """All patches of one level, resident on the device."""

    def __init__(self, spec: LevelSpec, boxes, M: int, device: torch.device,
                 stream: torch.cuda.Stream, need_gown: bool, owned: Optional[np.ndarray] = None,
                 gidx: Optional[np.ndarray] = None):
        """``owned`` (bool per patch) restricts stepping, filling, flagging and
        reductions to this rank's patches in a sharded run (the others are
        shadows, distributed.py); ``gidx`` = global indices of the patches."""
        self.spec = spec
        self.M = M
        self.device = device
        self.stream = stream
        b = np.asarray(boxes, dtype=np.int64).reshape(-1, 4)
        self.boxes = b
        self.P = len(b)
        self.gidx = np.arange(self.P, dtype=np.int64) if gidx is None else np.asarray(gidx, np.int64)
        self.owned = None if owned is None else np.asarray(owned, bool)
        nx = b[:, 2] - b[:, 0] + 1
        ny = b[:, 3] - b[:, 1] + 1
        cells = nx * ny
        self.ncells = int(cells.sum() if self.owned is None else cells[self.owned].sum())
        size = (nx + 2 * GHOST_WIDTH) * (ny + 2 * GHOST_WIDTH)
        aligned = (size + ALIGN - 1) // ALIGN * ALIGN
        self.offsets = np.concatenate([[0], np.cumsum(aligned)[:-1]]).astype(np.int64) if self.P else \
            np.zeros(0, np.int64)
        self.FS = max(int(aligned.sum()), ALIGN)
        self.max_cells = int(size.max()) if self.P else 0
        self.max_interior = int((nx * ny).max()) if self.P else 0
        import time as _t
        _p = POOL_PROF
        _t0 = _t.perf_counter()
        with torch.cuda.stream(stream):
            self.buf = [acquire(3 * M * self.FS, torch.float64, device, stream),
                        acquire(3 * M * self.FS, torch.float64, device, stream)]
            self.bathy = acquire(self.FS, torch.float64, device, stream)
            _t1 = _t.perf_counter()
            _p["acquire"] += _t1 - _t0
            for t in (self.buf[0], self.buf[1], self.bathy):
                dmemset(t, 0, stream)
            _t2 = _t.perf_counter()
            _p["zero"] += _t2 - _t1
            A = arena()
            self.box_d = A.upload(b.astype(np.int32), device, stream)
            self.off_d = A.upload(self.offsets, device, stream)
            _t3 = _t.perf_counter()
            _p["upload"] += _t3 - _t2
            self.tile_shape = N.step_tile(int((b[:, 2] - b[:, 0] + 1).max()) if self.P else 0, M)
            self.tile_tx = self.tile_shape[1]
            # the step work list is built on first use (tiles_d & co. below):
            # a regrid then enqueues its fill kernels without waiting for it
            self._tiles = None
            self.owned_d = None
            self.n_owned = self.P
            if self.owned is not None:
                ol = np.flatnonzero(self.owned).astype(np.int32)
                self.n_owned = len(ol)
                self.owned_d = A.upload(ol, device, stream) if len(ol) else dzeros(1, torch.int32, device, stream)
            self.speed_bits = dmemset(torch.empty(max(self.P, 1), dtype=torch.int64, device=device), 0xFF, stream)
            mapn = (spec.nx + 2 * GHOST_WIDTH) * (spec.ny + 2 * GHOST_WIDTH)
            _t4 = _t.perf_counter()
            self.own = dmemset(acquire(mapn, torch.int32, device, stream), 0xFF, stream)
            self.gown = dmemset(acquire(mapn, torch.int32, device, stream), 0xFF, stream) if need_gown else None
            _p["maps"] += _t.perf_counter() - _t4
        self.child: Optional[torch.Tensor] = None   # finer level's coarsened owner map
        self.cur = 0
        self.ghosts_in_cur = False
        self.time = 0.0
        L = N.lib()
        sh = _stream_handle(stream)
        if self.P:
            N.check(L.mlamr_paint_owner(self.own.data_ptr(), spec.nx, spec.ny, self.box_d.data_ptr(),
                                        self.P, 0, 0, 1, 1, self.max_interior, sh), "paint own")
            if self.gown is not None:
                N.check(L.mlamr_paint_owner(self.gown.data_ptr(), spec.nx, spec.ny, self.box_d.data_ptr(),
                                            self.P, GHOST_WIDTH, 1, 1, 1, self.max_cells, sh), "paint gown")

    # -- step work list (built lazily) ------------------------------------------
    def _build_tiles(self) -> None:
        import time as _t
        t0 = _t.perf_counter()
        tl = tile_list(self.boxes, self.tile_shape)
        if self.owned is not None and len(tl):
            tl = tl[self.owned[tl[:, 0]]]
        with torch.cuda.stream(self.stream):
            td = arena().upload(tl, self.device, self.stream) if len(tl) else \
                dzeros(3, torch.int32, self.device, self.stream)
            acc = dzeros(max(len(tl), 1) * (self.M + 2), torch.float64, self.device, self.stream)
        self._tiles = (tl, len(tl), td, acc)
        POOL_PROF["tile_list"] += _t.perf_counter() - t0

    def reorder_tiles(self, order: np.ndarray) -> None:
        """Permute the step work list (per-tile partials follow the list)."""
        if self._tiles is None:
            self._build_tiles()
        tl, n, _, acc = self._tiles
        tl = np.ascontiguousarray(tl[np.asarray(order, np.int64)])
        with torch.cuda.stream(self.stream):
            td = arena().upload(tl, self.device, self.stream) if len(tl) else \
                dzeros(3, torch.int32, self.device, self.stream)
        self._tiles = (tl, n, td, acc)

    @property
    def tiles(self) -> np.ndarray:
        if self._tiles is None:
            self._build_tiles()
        return self._tiles[0]

    @property
    def n_tiles(self) -> int:
        if self._tiles is None:
            self._build_tiles()
        return self._tiles[1]

    @property
    def tiles_d(self) -> torch.Tensor:
        if self._tiles is None:
            self._build_tiles()
        return self._tiles[2]

    @property
    def tile_acc(self) -> torch.Tensor:
        if self._tiles is None:
            self._build_tiles()
        return self._tiles[3]

    def release(self) -> None:
        """Hand the big buffers back for reuse by a later pool."""
        for t in (self.buf[0], self.buf[1], self.bathy, self.own, self.gown):
            if t is not None:
                release(t)
        self.buf = [None, None]
        self.bathy = None

    # -- views ---------------------------------------------------------------
    @property
    def state(self) -> torch.Tensor:
        return self.buf[self.cur]

    @property
    def other(self) -> torch.Tensor:
        return self.buf[1 - self.cur]

    def struct(self, state: Optional[torch.Tensor] = None) -> N.Level:
        s = self.spec
        lv = N.Level()
        lv.num_patches = self.P
        lv.num_layers = self.M
        lv.level_nx = s.nx
        lv.level_ny = s.ny
        lv.dx = s.dx
        lv.dy = s.dy
        lv.field_stride = self.FS
        lv.box = self.box_d.data_ptr()
        lv.offset = self.off_d.data_ptr()
        lv.state = (self.state if state is None else state).data_ptr()
        lv.bathy = self.bathy.data_ptr()
        lv.own = self.own.data_ptr()
        lv.gown = self.gown.data_ptr() if self.gown is not None else None
        return lv

    def ghost_plan(self):
        """Per-layout K2 plan (mlamr_ghost_plan): sibling source of every ghost
        cell, the compacted list of cells to interpolate from the parent, and
        the patches that need physical BCs -- restricted to owned patches."""
        if getattr(self, "_plan", None) is not None:
            return self._plan
        b = self.boxes
        nx = b[:, 2] - b[:, 0] + 1
        ny = b[:, 3] - b[:, 1] + 1
        ng = 4 * (nx + 2 * GHOST_WIDTH) + 4 * ny
        gbase = np.concatenate([[0], np.cumsum(ng)[:-1]]).astype(np.int64)
        total = int(ng.sum())
        A = arena()
        with torch.cuda.stream(self.stream):
            gbase_d = A.upload(gbase, self.device, self.stream)
            plan = torch.empty(max(total, 1), dtype=torch.int64, device=self.device)
            N.check(N.lib().mlamr_ghost_plan(self.struct(), gbase_d.data_ptr(), plan.data_ptr(), int(ng.max()),
                                             self.stream.cuda_stream), "ghost_plan")
            # interpolated cells (-1) compacted on the device: no host
            # round trip for their count (n_cells is the list's capacity)
            cap = max(total, 1)
            cells = torch.empty(2 * cap, dtype=torch.int32, device=self.device)
            count = dzeros(1, torch.int32, self.device, self.stream)
            if self.owned is not None:
                pl, nl = (self.owned_d.data_ptr(), self.n_owned) if self.n_owned else (None, 0)
            else:
                pl, nl = None, self.P
            if nl:
                N.check(N.lib().mlamr_plan_interp_cells(self.struct(), gbase_d.data_ptr(), plan.data_ptr(), pl,
                                                        nl, int(ng.max()), cells.data_ptr(), count.data_ptr(),
                                                        self.stream.cuda_stream), "plan_interp_cells")
            self.interp_count = count
        s = self.spec
        touch = (b[:, 0] == 0) | (b[:, 2] == s.nx - 1) | (b[:, 1] == 0) | (b[:, 3] == s.ny - 1)
        if self.owned is not None:
            touch &= self.owned
        bcp = np.flatnonzero(touch).astype(np.int32)
        bc_d = A.upload(bcp, self.device, self.stream) if len(bcp) else dzeros(1, torch.int32, self.device,
                                                                                self.stream)
        self._plan = (gbase_d, plan, cells, cap if nl else 0, bc_d, len(bcp), int(ng.max()) if len(ng) else 0)
        return self._plan

    def coarse_base(self, rx: int, ry: int):
        """(device int64 prefix sums of the coarse cells under each patch,
        total) for the flat average_down.  All local patches: under
        sharding the coarse owner averages the children it holds as
        shadows (delivered whole by the pre-coarsening refresh)."""
        key = (rx, ry)
        cache = getattr(self, "_cbase", None)
        if cache is None or cache[0] != key:
            b = self.boxes
            n = ((b[:, 2] - b[:, 0] + 1) // rx) * ((b[:, 3] - b[:, 1] + 1) // ry) if self.P else np.zeros(0, np.int64)
            base = np.concatenate([[0], np.cumsum(n)]).astype(np.int64)
            with torch.cuda.stream(self.stream):
                d = arena().upload(base, self.device, self.stream)
            cache = (key, d, int(base[-1]))
            self._cbase = cache
        return cache[1], cache[2]

    def copy_pairs(self):
        """(device int64 [n, 2] (destination, source) offsets, n): the sibling
        copies of the ghost fill for the owned patches (built once per layout)."""
        if getattr(self, "_pairs", None) is not None:
            return self._pairs
        gbase_d, plan = self.ghost_plan()[:2]
        b = self.boxes
        ng = 4 * (b[:, 2] - b[:, 0] + 1 + 2 * GHOST_WIDTH) + 4 * (b[:, 3] - b[:, 1] + 1)
        A = arena()
        lst = np.flatnonzero(self.owned) if self.owned is not None else np.arange(self.P)
        if len(lst):
            lbase = np.concatenate([[0], np.cumsum(ng[lst])[:-1]]).astype(np.int64)
            ltot = int(ng[lst].sum())
            with torch.cuda.stream(self.stream):
                pl_d = A.upload(lst.astype(np.int32), self.device, self.stream)
                lb_d = A.upload(lbase, self.device, self.stream)
                raw = torch.empty(2 * ltot, dtype=torch.int64, device=self.device)
                N.check(N.lib().mlamr_copy_pairs_of_plan(self.struct(), gbase_d.data_ptr(), plan.data_ptr(),
                                                         pl_d.data_ptr(), len(lst), lb_d.data_ptr(),
                                                         int(ng.max()), raw.data_ptr(), self.stream.cuda_stream),
                        "copy_pairs_of_plan")
                raw = raw.view(-1, 2)
                pairs = raw[raw[:, 0] >= 0].contiguous()
            self._pairs = (pairs, int(pairs.shape[0]))
        else:
            self._pairs = (torch.zeros(2, dtype=torch.int64, device=self.device), 0)
        return self._pairs

    def work_list(self):
        """(device patch-list pointer, count) of the patches this rank owns,
        or (None, 0) when it owns them all (single-GPU runs)."""
        if self.owned_d is None:
            return None, 0
        return self.owned_d.data_ptr(), self.n_owned

    def local_of(self, g: np.ndarray) -> np.ndarray:
        """Local indices of global patch indices (all must be held)."""
        return np.searchsorted(self.gidx, g)

    def copy_segments(self, src_buf, src_stride, dst_buf, dst_stride, src_off, dst_off, sizes,
                      stream: Optional[torch.cuda.Stream] = None) -> None:
        """Whole-block copies of all 3M planes (multi-GPU shadow exchange),
        on ``stream`` (default: the pool's)."""
        n = len(sizes)
        if n == 0:
            return
        st = stream or self.stream
        seg = np.stack([np.asarray(src_off, np.int64), np.asarray(dst_off, np.int64),
                        np.asarray(sizes, np.int64)], axis=1)
        seg_d = arena().upload(seg, self.device, st)
        N.check(N.lib().mlamr_copy_segments(src_buf.data_ptr(), int(src_stride), dst_buf.data_ptr(),
                                            int(dst_stride), seg_d.data_ptr(), n, int(np.max(sizes)),
                                            3 * self.M, st.cuda_stream), "copy_segments")

    def blocks_per_patch(self, cells: int) -> int:
        return int(max(1, min(64, (cells + NTHREADS - 1) // NTHREADS)))

    # -- host transfer (frames, flags, tests) ----------------------------------
    def patch_arrays(self, p: int, which: Optional[torch.Tensor] = None, host: Optional[np.ndarray] = None):
        """(h, hu, hv, bathy) numpy arrays [M, NY, NX] of patch p."""
        lo_i, lo_j, hi_i, hi_j = self.boxes[p]
        NX = hi_i - lo_i + 1 + 2 * GHOST_WIDTH
        NY = hi_j - lo_j + 1 + 2 * GHOST_WIDTH
        off = int(self.offsets[p])
        if host is None:
            host = self.download(which)
        st, bathy = host
        M = self.M
        blk = st[:, off:off + NX * NY].reshape(3 * M, NY, NX)
        return (blk[:M].copy(), blk[M:2 * M].copy(), blk[2 * M:].copy(),
                bathy[off:off + NX * NY].reshape(NY, NX).copy())

    def download(self, which: Optional[torch.Tensor] = None):
        t = self.state if which is None else which
        torch.cuda.current_stream().wait_stream(self.stream)
        st = t.view(3 * self.M, self.FS).cpu().numpy()
        return st, self.bathy.cpu().numpy()

    def upload_patches(self, arrays, which: Optional[torch.Tensor] = None, bathy: bool = False) -> None:
        """arrays[p] = (h, hu, hv) [M, NY, NX] (or a bathymetry [NY, NX])."""
        M = self.M
        if bathy:
            host = np.zeros(self.FS)
        else:
            host = np.zeros((3 * M, self.FS))
        for p, arr in enumerate(arrays):
            off = int(self.offsets[p])
            if bathy:
                host[off:off + arr.size] = arr.ravel()
            else:
                h, hu, hv = arr
                n = h[0].size
                for m in range(M):
                    host[m, off:off + n] = h[m].ravel()
                    host[M + m, off:off + n] = hu[m].ravel()
                    host[2 * M + m, off:off + n] = hv[m].ravel()
        t = torch.from_numpy(host.reshape(-1))
        with torch.cuda.stream(self.stream):
            if bathy:
                self.bathy.copy_(t)
            else:
                (self.state if which is None else which).copy_(t)


def empty_level_struct(spec: LevelSpec, M: int) -> N.Level:
    """A level with no patches (owner maps NULL: every lookup misses)."""
    lv = N.Level()
    lv.num_patches = 0
    lv.num_layers = M
    lv.level_nx = spec.nx
    lv.level_ny = spec.ny
    lv.dx = spec.dx
    lv.dy = spec.dy
    lv.field_stride = 0
    lv.box = None
    lv.offset = None
    lv.state = None
    lv.bathy = None
    lv.own = None
    lv.gown = None
    return lv


def paint_child_map(parent_spec: LevelSpec, fine_boxes: np.ndarray, rx: int, ry: int,
                    device, stream) -> torch.Tensor:
    """Owner map, in the parent's index space, of the fine boxes' coarse
    footprints (coverage_mask, mesh.py:271-279)."""
    mapn = (parent_spec.nx + 2 * GHOST_WIDTH) * (parent_spec.ny + 2 * GHOST_WIDTH)
    with torch.cuda.stream(stream):
        m = dmemset(acquire(mapn, torch.int32, device, stream), 0xFF, stream)
        if len(fine_boxes):
            bd = arena().upload(np.asarray(fine_boxes, np.int32).reshape(-1, 4), device, stream)
            nx = fine_boxes[:, 2] - fine_boxes[:, 0] + 1
            ny = fine_boxes[:, 3] - fine_boxes[:, 1] + 1
            mc = int(((nx // rx) * (ny // ry)).max())
            N.check(N.lib().mlamr_paint_owner(m.data_ptr(), parent_spec.nx, parent_spec.ny, bd.data_ptr(),
                                              len(fine_boxes), 0, 0, rx, ry, mc, stream.cuda_stream),
                    "paint child")
            m._keep = bd  # keep the box tensor alive until the stream passes
    return m
