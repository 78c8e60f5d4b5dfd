"""Subcycled multi-level driver on the device (driver.py:89-362 under
/root/reference/pkg/src/mlamr).

The recursion, host scalars (dt, theta, r_t, times) and flag clustering
stay in Python exactly as the reference orders them; every per-patch loop
of the reference is replaced by one level-batched kernel launch through the
C-ABI:

========================================  =====================================
reference                                 here
========================================  =====================================
``_step_patches`` -> ``step_patch`` xP    ``mlamr_step`` + ``mlamr_step_finalize``
``fill_level_ghosts`` -> ``fill_ghosts``  ``mlamr_fill_ghosts``
stash copies (driver.py:260-264)          the step's untouched source buffer
``average_down``                          ``mlamr_average_down``
``rebuild_child_level`` data movement     ``mlamr_regrid_fill`` / ``_derefine_delta``
``flag_cells`` per-cell tests             ``mlamr_flag_cells``
``stable_dt`` / dynamic r_t speeds        ``mlamr_max_speed_tiles``
``composite_mass`` + ``_check_finite``    ``mlamr_level_reduce``
========================================  =====================================

Host/device synchronisation happens once per coarse step (dt, status,
composite mass) plus once per regrid (flag map).
"""

from __future__ import annotations

import copy
import ctypes
import os
import time
from collections import defaultdict
from contextlib import contextmanager
from dataclasses import asdict, dataclass, field, fields, replace

import numpy as np
import torch

from . import _native as N
from .device import LevelPool, acquire, arena, dmemset, dzeros, empty_level_struct, paint_child_map, release
from .errors import CflViolationError, NumericalAbortError, TimeSyncError, raise_status
from .mesh import GHOST_WIDTH, IndexBox, LevelSpec, boxes_array, paint
from .regrid import chop_boxes, cluster_boxes, cluster_boxes_device, nesting_allowed
from .problems import gradient_flags_map

_TIME_RTOL = 1e-12
_LOG_STEP_BYTES = bool(__import__("os").environ.get("MLAMR_LOG_STEP_BYTES"))


@dataclass
class RunStats:
    """Counters and timers of one run (driver.py:44-78): same fields and
    the same ``to_json`` layout as the reference's stats.json."""
    wall_time: float = 0.0
    cpu_time: float = 0.0
    total_cell_updates: int = 0
    cell_updates_per_level: dict = field(default_factory=dict)
    num_coarse_steps: int = 0
    num_regrids: int = 0
    workers: int = 1
    amr_enabled: bool = True
    initial_mass: list = field(default_factory=list)
    final_mass: list = field(default_factory=list)
    mass_drift: list = field(default_factory=list)
    refine_delta: list = field(default_factory=list)
    derefine_delta: list = field(default_factory=list)
    sync_delta: list = field(default_factory=list)
    hyperbolicity_warnings: int = 0
    wet_prefix_repairs: int = 0
    clipped_mass: list = field(default_factory=list)

    @classmethod
    def from_json(cls, path) -> "RunStats":
        import json
        with open(path) as f:
            data = json.load(f)
        data["cell_updates_per_level"] = {int(k): int(v) for k, v in data.get("cell_updates_per_level", {}).items()}
        known = {f.name for f in fields(cls)}
        return cls(**{k: v for k, v in data.items() if k in known})

    def to_json(self, path) -> None:
        import json
        data = asdict(self)
        data["cell_updates_per_level"] = {str(k): int(v) for k, v in self.cell_updates_per_level.items()}
        with open(path, "w") as f:
            json.dump(data, f, indent=2, sort_keys=True, default=lambda o: o.item() if hasattr(o, "item") else str(o))
            f.write("\n")


def regrid_fill_bytes(new_boxes, old_boxes, rx: int, ry: int, M: int) -> int:
    """Algorithmic bytes of one k_regrid_fill launch (SURVEY.md §8(d) K3 +
    K5): 8*(3M + 1 + (3M+1)/(r_x r_y)) per refined fine cell (written state,
    read bathymetry, the parent stencil amortised over its children) and
    8*6M per cell copied from an old patch.  Both box sets are
    ratio-aligned, so the overlap is counted on the coarse grid."""
    nb = np.asarray(new_boxes, np.int64).reshape(-1, 4)
    ob = np.asarray(old_boxes, np.int64).reshape(-1, 4)
    total = int(((nb[:, 2] - nb[:, 0] + 1) * (nb[:, 3] - nb[:, 1] + 1)).sum())
    copied = 0
    if len(ob) and len(nb):
        c_new = np.stack([nb[:, 0] // rx, nb[:, 1] // ry, (nb[:, 2] + 1) // rx, (nb[:, 3] + 1) // ry], 1)
        c_old = np.stack([ob[:, 0] // rx, ob[:, 1] // ry, (ob[:, 2] + 1) // rx, (ob[:, 3] + 1) // ry], 1)
        W = int(max(c_new[:, 2].max(), c_old[:, 2].max())) + 1
        H = int(max(c_new[:, 3].max(), c_old[:, 3].max())) + 1
        d = np.zeros((H + 1, W + 1), np.int32)
        np.add.at(d, (c_old[:, 1], c_old[:, 0]), 1)
        np.add.at(d, (c_old[:, 1], c_old[:, 2]), -1)
        np.add.at(d, (c_old[:, 3], c_old[:, 0]), -1)
        np.add.at(d, (c_old[:, 3], c_old[:, 2]), 1)
        cov = (np.cumsum(np.cumsum(d, 0), 1) > 0).astype(np.int64)
        sat = np.zeros((H + 2, W + 2), np.int64)
        sat[1:, 1:] = np.cumsum(np.cumsum(cov, 0), 1)
        x0, y0, x1, y1 = c_new.T
        copied = int((sat[y1, x1] - sat[y0, x1] - sat[y1, x0] + sat[y0, x0]).sum()) * rx * ry
    refined = total - copied
    return int(8 * (3 * M + 1 + (3 * M + 1) / (rx * ry)) * refined + 8 * 6 * M * copied)


def _pinned_bathy(problem) -> list:
    """The problem's per-level bathymetry arrays staged once in pinned host
    memory (cached on the problem object, keyed by the arrays' identity), so
    every Simulation built from the problem -- including restores from a
    snapshot -- uploads them as asynchronous DMA instead of pageable copies."""
    key = tuple(id(b) for b in problem.bathy_levels)
    cached = getattr(problem, "_bathy_pinned", None)
    if cached is None or cached[0] != key:
        pins = []
        for b in problem.bathy_levels:
            a = np.ascontiguousarray(b, dtype=np.float64)
            t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
            t.numpy()[...] = a
            pins.append(t)
        cached = (key, pins)
        problem._bathy_pinned = cached
    return cached[1]


class Simulation:
    """Device-resident counterpart of driver.Simulation over a harness problem
    (:mod:`paper_1803_01450_b200.problems`)."""

    def __init__(self, problem, device: str = "cuda", stream: torch.cuda.Stream | None = None,
                 _restore: dict | None = None, reserve_factor: float = 2.0):
        """``reserve_factor``: after the initial hierarchy is built, warm the
        device allocator with that multiple of its buffer bytes, so pools
        that grow at regrids do not pay cudaMalloc inside the time loop
        (device.reserve).  A pool that outgrows its recycled buffers asks for
        1.5x its size in one piece (~6.6 GB for C4's finest level); with a
        factor of 1 that request found the warmed block already split in
        some runs and cost an ~80 ms cudaMalloc inside the loop (4 ms per
        coarse step of a 20-step bench), hence 2."""
        self._common_init(problem, device, stream)
        if _restore is not None:
            self._restore_from(_restore)
        else:
            base = self._new_pool(1, self.level1_boxes())
            self._set_initial(base)
            self.levels[1] = base
            for lev in range(1, self.L):
                self._rebuild(lev, init=True)
            self._mass_prev = self.composite_mass()
            self.stats.initial_mass = list(self._mass_prev)
            self._sync_status("building the initial hierarchy")
        if reserve_factor > 0:
            from .device import reserve
            reserve(int(reserve_factor * self.device_bytes()), self.dev, self.stream)

    def level1_boxes(self, default_tile: int = 0) -> np.ndarray:
        """Level 1's patches: the reference's single patch over the domain
        (mesh.py:372-375), or -- ``MLAMR_L1_TILE=T`` -- aligned T x T tiles
        of it.  Tiling is bit-exact (SURVEY.md App. C probe 4: a tile's halo
        is its siblings' interior at the same time level, the domain edge's
        ghost cells the same boundary conditions;
        tests/test_gpu_driver.py::test_tiled_level1_is_bit_identical) and is
        what lets a sharded run spread level 1 over the ranks instead of
        giving it to rank 0."""
        nx, ny = self.specs[0].nx, self.specs[0].ny
        full = boxes_array([IndexBox(0, 0, nx - 1, ny - 1)])
        T = int(os.environ.get("MLAMR_L1_TILE") or default_tile)
        if T <= 0 or (T >= nx and T >= ny):
            return full
        from .regrid import chop_boxes
        return np.asarray(chop_boxes(full, T, T, aligned=True), dtype=np.int64).reshape(-1, 4)

    def device_bytes(self) -> int:
        """Bytes of the level pools' state and bathymetry buffers."""
        n = 0
        for pool in self.levels.values():
            for t in list(getattr(pool, "buf", [])) + [getattr(pool, "bathy", None)]:
                if t is not None:
                    n += t.numel() * t.element_size()
        return n

    def _common_init(self, problem, device, stream) -> None:
        self.lib = N.lib()
        self.pb = problem
        self.M = M = problem.num_layers
        self.prm = N.make_params(M, problem.densities, problem.gravity, problem.dry_tolerance)
        self.specs = [LevelSpec(*s) for s in problem.level_specs()]
        self.L = len(self.specs)
        self.bcs = N.bc_array(problem.boundaries)
        dev = torch.device(device)
        if dev.type == "cuda" and dev.index is None:   # recycled buffers compare devices exactly
            dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        self.stream = stream or torch.cuda.current_stream(self.dev)
        self.sh = self.stream.cuda_stream
        with torch.cuda.stream(self.stream):
            self.status = torch.zeros(1, dtype=torch.int32, device=self.dev)
            self.bad = torch.full((1,), 2 ** 31 - 1, dtype=torch.int32, device=self.dev)
            self.acc = torch.zeros(M + 2, dtype=torch.float64, device=self.dev)
            self.delta_acc = torch.zeros(3, M, dtype=torch.float64, device=self.dev)  # refine, derefine, event
            self._mass_d = torch.zeros(M, dtype=torch.float64, device=self.dev)
            # whole-level bathymetry (the scenario's fill_bathymetry source):
            # async copies from pinned host staging kept on the problem
            self.level_bathy = [b.to(self.dev, non_blocking=True) for b in _pinned_bathy(problem)]
            self.scratch = torch.zeros(1, dtype=torch.float64, device=self.dev)
            self._eta_rest = torch.tensor(list(problem.eta_rest), dtype=torch.float64, device=self.dev)
            self._wave_tol = torch.tensor(list(problem.wave_tolerance), dtype=torch.float64, device=self.dev)
        self._flagbuf = {}
        self._scratch_bufs = {}
        self._pinned_bufs = {}
        # the step's per-patch observed speeds are reset to -1 by its
        # finalize; True keeps them readable after the step (tests)
        self.keep_step_speeds = False
        # {name: [(start event, end event, algorithmic bytes)]} when not None
        self.kernel_timer = None
        self._speed_cache = None   # (state key, level-1 speed bits) from _step_readback
        self._restores = 0
        # childless levels: sibling ghost copy inside the step's staging
        # (mlamr_step with a ghost plan; the finite check then reads those
        # cells through the plan too).  On C4 it drops the 0.29 ms sibling
        # copy per finest fill for ~0.19 ms of plan lookups per step launch
        # (issued behind the tile's other loads): 70.9 -> 68.7 ms per coarse
        # step.  MLAMR_FUSE_SIBLING=0 restores the separate copy.
        self.fuse_sibling_fill = os.environ.get("MLAMR_FUSE_SIBLING", "1") == "1"
        self.levels: dict[int, LevelPool] = {}
        self.steps = {s.level: 0 for s in self.specs}
        self._stash = {}
        self.stats = RunStats()
        self.time = 0.0
        self.launches = 0
        self.d2h_bytes = 0
        self.h2d_bytes = sum(b.numel() * 8 for b in self.level_bathy)
        self.step_timer_level = None   # record CUDA events around this level's step kernel
        self.step_events = []
        self.host_prof = defaultdict(float)   # host wall seconds per phase (incl. syncs)

    # -- helpers ----------------------------------------------------------------
    @contextmanager
    def _timed(self, name: str):
        t0 = time.perf_counter()
        try:
            yield
        finally:
            self.host_prof[name] += time.perf_counter() - t0

    def _scratch(self, name: str, n: int, zero: bool = True) -> torch.Tensor:
        """A float64 device buffer of >= n elements kept across calls (grown
        by half when too small): per-block partial sums are allocated every
        step and regrid, and fresh allocations there occasionally reached
        cudaMalloc inside the time loop.  Reuse is ordered on the stream."""
        buf = self._scratch_bufs.get(name)
        if buf is None or buf.numel() < n:
            with torch.cuda.stream(self.stream):
                buf = torch.empty(max(int(n * 1.5), 1024), dtype=torch.float64, device=self.dev)
            self._scratch_bufs[name] = buf
        out = buf[:max(n, 1)]
        if zero:
            dmemset(out, 0, self.stream)
        return out

    def spec(self, level: int) -> LevelSpec:
        return self.specs[level - 1]

    def _call(self, fn, *args, what=""):
        what = what or fn.__name__
        self.launches += 2 if what == "mlamr_step" else 1   # + k_make_desc
        N.check(fn(*args), what)

    # -- per-kernel timing for the bench (CUDA events on the driver stream) ------
    def _kt0(self):
        """Start event of a timed launch, or None when timing is off."""
        if self.kernel_timer is None:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record(self.stream)
        return e

    def _kt1(self, name: str, e0, nbytes) -> None:
        """End of a timed launch: ``nbytes`` (int or a callable evaluated
        after the timed region) = its algorithmic HBM bytes."""
        if e0 is None:
            return
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(self.stream)
        self.kernel_timer.setdefault(name, []).append((e0, e1, nbytes))

    def _new_pool(self, level: int, boxes: np.ndarray) -> LevelPool:
        pool = LevelPool(self.spec(level), boxes, self.M, self.dev, self.stream, need_gown=level < self.L)
        if pool.P:
            self._call(self.lib.mlamr_fill_bathymetry, pool.struct(), self.level_bathy[level - 1].data_ptr(),
                       self.bcs, self.sh)
            if level > 1 and level - 1 in self.levels:
                self._check_bathymetry(pool, self.levels[level - 1], self.spec(level - 1))
        return pool

    def _check_bathymetry(self, fine: LevelPool, coarse: LevelPool, cs: LevelSpec) -> None:
        """check_bathymetry_consistency (coarsen.py:79-100) for every new
        fine patch against the coarse interiors, on the device; a violation
        sets MLAMR_ST_BATHY, raised as the reference's AssertionError at the
        next status check (the end of this coarse step, or construction)."""
        if coarse.P == 0:
            return
        cbase, n = fine.coarse_base(cs.r_x, cs.r_y)
        self._call(self.lib.mlamr_check_bathymetry, fine.struct(), coarse.struct(), cs.r_x, cs.r_y, 1e-12,
                   cbase.data_ptr(), n, self.status.data_ptr(), self.bad.data_ptr(), self.sh)

    def _set_initial(self, pool: LevelPool) -> None:
        """Evaluate the problem's initial condition once per band of patches
        sharing the same rows (the evaluators are cellwise, so slicing a band
        equals evaluating each patch box) and upload it."""
        g = GHOST_WIDTH
        arrays = [None] * pool.P
        bands = {}
        for p, b in enumerate(pool.boxes):
            bands.setdefault((int(b[1]), int(b[3])), []).append(p)
        for (lo_j, hi_j), members in bands.items():
            lo_i = int(min(pool.boxes[p][0] for p in members)) - g
            hi_i = int(max(pool.boxes[p][2] for p in members)) + g
            h, hu, hv = self.pb.initial_state_box(pool.spec.level, (lo_i, lo_j - g, hi_i, hi_j + g))
            for p in members:
                a = int(pool.boxes[p][0]) - g - lo_i
                w = int(pool.boxes[p][2] - pool.boxes[p][0]) + 1 + 2 * g
                arrays[p] = (h[:, :, a:a + w], hu[:, :, a:a + w], hv[:, :, a:a + w])
        pool.upload_patches(arrays)

    def _sync_status(self, where: str = "") -> None:
        self.d2h_bytes += 4
        # the status word is written on the driver stream, which need not
        # be the caller's current stream (torch streams are non-blocking)
        self.stream.synchronize()
        st = int(self.status.item())
        if st:
            bad = int(self.bad.item())
            if st & N.ST_CFL:
                raise CflViolationError(f"Courant number > 1 on patch {bad} {where}")
            raise_status(st, where)

    # -- mass accounting and finite check (driver.py:138-153, 286-297) ---------
    def _level_reduce(self, level: int, tot: torch.Tensor, init: bool) -> None:
        """Adds this level's composite volume per layer into ``tot`` (or
        sets it, ``init``) and runs the finite check (status)."""
        pool = self.levels[level]
        if pool.P == 0:
            if init:
                self._call(self.lib.mlamr_sum_partials, None, 0, self.M, 1.0, tot.data_ptr(), None, 1, self.sh)
            return
        # a few blocks per patch, each thread over ~8 cells: the per-block
        # reduction, not the bytes, had dominated with one cell per thread
        # (up to 1024 blocks for a level of a few large patches, e.g. a
        # 1280^2 level 1: 64 blocks left most of the GPU idle)
        cap = 64 if pool.P >= 64 else 1024
        bpp = max(1, min(cap, -(-pool.max_cells // (8 * 256))))
        with torch.cuda.stream(self.stream):
            part = self._scratch("reduce", pool.P * bpp * self.M)
            ghosts = pool.state if pool.ghosts_in_cur else pool.other
            child = pool.child.data_ptr() if pool.child is not None else None
            pl, nl = pool.work_list()
            gb = gp = None
            if getattr(pool, "fused_frame", False) and not pool.ghosts_in_cur:
                gbase, plan = pool.ghost_plan()[:2]
                gb, gp = gbase.data_ptr(), plan.data_ptr()
            e0 = self._kt0()
            self._call(self.lib.mlamr_level_reduce_planned, pool.struct(), pool.state.data_ptr(),
                       ghosts.data_ptr(), child, part.data_ptr(), bpp, self.status.data_ptr(), pl, nl, gb, gp,
                       self.sh)
            # K6: every state value of every patch, ghost frames included (finite check)
            self._kt1(f"k_level_reduce L{level}", e0, 8 * 3 * self.M * pool.FS)
            s = self.spec(level)
            self._call(self.lib.mlamr_sum_partials, part.data_ptr(), pool.P * bpp, self.M, s.dx * s.dy,
                       tot.data_ptr(), None, int(init), self.sh)

    def _mass_device(self) -> torch.Tensor:
        """Composite volume per layer on the device (driver.py:138-153)."""
        tot = self._mass_d
        first = True
        for lev in range(1, self.L + 1):
            if lev in self.levels:
                self._level_reduce(lev, tot, first)
                first = False
        return tot

    def _pinned(self, name: str, n: int, dtype) -> torch.Tensor:
        key = (name, dtype)
        buf = self._pinned_bufs.get(key)
        if buf is None or buf.numel() < n:
            buf = torch.empty(max(2 * n, 64), dtype=dtype, pin_memory=True)
            self._pinned_bufs[key] = buf
        return buf[:n]

    def composite_mass(self) -> np.ndarray:
        with torch.cuda.stream(self.stream):
            tot = self._mass_device()
            out = self._pinned("mass", self.M, torch.float64)
            out.copy_(tot, non_blocking=True)
        self.stream.synchronize()
        arena().reset()
        self.d2h_bytes += 8 * self.M
        return out.numpy().copy()

    # -- ghost filling (driver.py:157-190) ------------------------------------
    def fill_level_ghosts(self, level: int, t: float, siblings: bool = True, part: str = "all") -> None:
        """Ghost frames of a level at time t (driver.py:175-190).  With
        ``siblings=False`` the sibling copies are left to the step that
        follows (mlamr_step reads sibling halo cells through the ghost plan);
        only patches with physical BCs get them, because their BC corners
        read the copied frame.  ``part`` (with siblings=False) splits that
        fill: "interp" = the parent-interpolated cells only, "bc" = the BC
        patches' sibling copies and boundary conditions only (the sharded
        driver runs them on either side of a shadow exchange)."""
        pool = self.levels[level]
        if pool.P == 0:
            return
        if level == 1:
            par_ptr, old_ptr, theta, rx, ry = None, None, 0.0, 1, 1
        else:
            par = self.levels[level - 1]
            ps = self.spec(level - 1)
            rx, ry = ps.r_x, ps.r_y
            par_struct = par.struct()
            par_ptr = ctypes.byref(par_struct)
            old_ptr, theta = None, 0.0
            st = self._stash.get(level - 1)
            if st is not None:
                t0, dt, old = st
                theta = min(1.0, max(0.0, (t - t0) / dt)) if dt > 0 else 1.0
                old_ptr = old.data_ptr()
        gbase, plan, cells, n_cells, bc_d, n_bc, max_ghost = pool.ghost_plan()
        if siblings and max_ghost < 256:
            # small patches (fewer ghost cells than a block has threads):
            # the sibling copies as one flat gather/scatter, before the
            # planned fill (whose BC pass reads copied corner cells), which
            # then skips them
            pairs, n_pairs = pool.copy_pairs()
            self._call(self.lib.mlamr_fill_copy_pairs, pool.state.data_ptr(), pool.FS, pairs.data_ptr(), n_pairs,
                       self.M, self.status.data_ptr(), self.sh)
            pl, nl = bc_d.data_ptr(), 0
        elif siblings:
            pl, nl = pool.work_list()
        else:
            pl, nl = bc_d.data_ptr(), n_bc
        if not siblings and part == "interp":
            nl, n_bc = 0, 0
        elif not siblings and part == "bc":
            n_cells = 0
        timed = not siblings and level > 1 and n_cells
        e0 = self._kt0() if timed else None
        self._call(self.lib.mlamr_fill_ghosts_planned, pool.struct(), par_ptr, old_ptr, theta, rx, ry, self.bcs,
                   self.prm, self.status.data_ptr(), gbase.data_ptr(), plan.data_ptr(), pl, nl, max_ghost,
                   cells.data_ptr(), n_cells, pool.interp_count.data_ptr(), bc_d.data_ptr(), n_bc, self.sh)
        if e0 is not None:
            # K2 on a fused level: the parent-interpolated ghost cells (the
            # sibling copies run inside the step); per cell 3M written, the
            # bathymetry read, 2 x 3M parent values (old, new) amortised over
            # the r_x r_y children of a parent cell
            M = self.M
            self._kt1(f"k_fill_interp L{level}", e0,
                      lambda c=pool.interp_count, f=8 * (3 * M + 1 + 2 * 3 * M / (rx * ry)): int(f * int(c.item())))
        pool.ghosts_in_cur = True

    # -- regridding (driver.py:192-222, regrid.py:235-353) -------------------------
    def level_surfaces(self, level: int, layers) -> tuple:
        """Level-wide surfaces of the given layers and the covered mask (host)."""
        pool = self.levels[level]
        s = self.spec(level)
        eta = np.zeros((len(layers), s.ny, s.nx))
        covered = np.zeros((s.ny, s.nx), bool)
        host = pool.download()
        g = GHOST_WIDTH
        for p in range(pool.P):
            h, hu, hv, b = pool.patch_arrays(p, host=host)
            hi = h[:, g:-g, g:-g]
            e = np.cumsum(hi[::-1], axis=0)[::-1] + b[g:-g, g:-g]
            lo_i, lo_j, hi_i, hi_j = pool.boxes[p]
            eta[:, lo_j:hi_j + 1, lo_i:hi_i + 1] = e[list(layers)]
            covered[lo_j:hi_j + 1, lo_i:hi_i + 1] = True
        return eta, covered

    def _flag_buffers(self, level: int):
        s = self.spec(level)
        n = s.ny * s.nx
        key = (level, n)
        buf = self._flagbuf.get(key)
        if buf is None:
            with torch.cuda.stream(self.stream):
                buf = {
                    "bits": dzeros(n, torch.uint8, self.dev, self.stream),
                    "scratch": torch.empty(3 * n, dtype=torch.uint8, device=self.dev),
                    "flags": torch.empty(n, dtype=torch.uint8, device=self.dev),
                    "allowed": torch.empty(n, dtype=torch.uint8, device=self.dev),
                    "flags_h": torch.empty(n, dtype=torch.uint8, pin_memory=True),
                    "allowed_h": torch.empty(n, dtype=torch.uint8, pin_memory=True),
                }
            self._flagbuf[key] = buf
        return buf

    def flags_and_allowed(self, level: int):
        """Refinement flags of a level (already restricted to the nesting
        mask) and the nesting mask, as host uint8 maps [ny, nx]."""
        pool = self.levels[level]
        s = self.spec(level)
        rule = self.pb.flag_rule
        if self._device_rule():
            b = self._flag_buffers(level)
            self._device_flags(level)
            with torch.cuda.stream(self.stream):
                b["flags_h"].copy_(b["flags"], non_blocking=True)
                b["allowed_h"].copy_(b["allowed"], non_blocking=True)
            self.stream.synchronize()
            arena().reset()   # the stream is drained: staged uploads are complete
            self.d2h_bytes += 2 * s.ny * s.nx
            return (b["flags_h"].numpy().reshape(s.ny, s.nx).view(np.bool_),
                    b["allowed_h"].numpy().reshape(s.ny, s.nx).view(np.bool_))
        from .mesh import dilate
        covered = paint(pool.boxes, s.ny, s.nx)
        if rule[0] == "gradient":
            eta, covered = self.level_surfaces(level, rule[3])
            f = gradient_flags_map(eta, covered, s.dx, s.dy, rule[1])
            f = dilate(f, rule[2]) & covered
        elif rule[0] == "bernoulli":
            f = self.pb.bernoulli_flags(level, self.steps[level])
            f = dilate(f, rule[2]) & covered
        else:
            raise ValueError(rule)
        allowed = nesting_allowed(pool.boxes, s.ny, s.nx)
        region = self.pb.region_mask(level)
        if region is not None:
            allowed = allowed & region
        return f & allowed, allowed

    def flags_for(self, level: int) -> np.ndarray:
        return self.flags_and_allowed(level)[0]

    def _device_rule(self) -> bool:
        """Flag rules evaluated on the device: the reference rule, and the
        harness Bernoulli rule (its coverage comes from the level's owner
        map, which holds every patch on a single GPU)."""
        return self.pb.flag_rule[0] in ("reference", "bernoulli", "gradient")

    def _device_flags(self, level: int):
        """Flag rule + nesting mask on the device (0/1 byte maps)."""
        pool = self.levels[level]
        s = self.spec(level)
        b = self._flag_buffers(level)
        if self.pb.flag_rule[0] == "gradient":
            _, tol, width, layers = self.pb.flag_rule
            mask = 0
            for m in layers:
                mask |= 1 << int(m)
            key = ("eta", level)
            if key not in self._flagbuf:
                with torch.cuda.stream(self.stream):
                    self._flagbuf[key] = torch.empty(len(layers) * s.ny * s.nx, dtype=torch.float64,
                                                     device=self.dev)
            with torch.cuda.stream(self.stream):
                self._call(self.lib.mlamr_flags_gradient, pool.struct(), pool.state.data_ptr(), self.prm, mask,
                           float(tol), int(width), b["flags"].data_ptr(), b["allowed"].data_ptr(),
                           b["scratch"].data_ptr(), self._flagbuf[key].data_ptr(), self.sh)
                region = self._region_mask_d(level)
                if region is not None:
                    b["flags"].mul_(region)
                    b["allowed"].mul_(region)
            return b["flags"], b["allowed"]
        if self.pb.flag_rule[0] == "bernoulli":
            seed = int(self.pb.seed) & 0xFFFFFFFFFFFFFFFF
            sid = (1000 + 97 * level + 7919 * int(self.steps[level])) & 0xFFFFFFFFFFFFFFFF
            with torch.cuda.stream(self.stream):
                self._call(self.lib.mlamr_flags_bernoulli, pool.own.data_ptr(), s.ny, s.nx, seed, sid,
                           float(self.pb.bernoulli[0]), int(self.pb.flag_rule[2]), b["flags"].data_ptr(),
                           b["allowed"].data_ptr(), b["scratch"].data_ptr(), self.sh)
                region = self._region_mask_d(level)
                if region is not None:
                    b["flags"].mul_(region)
                    b["allowed"].mul_(region)
            return b["flags"], b["allowed"]
        with torch.cuda.stream(self.stream):
            dmemset(b["bits"], 0, self.stream)
            pl, nl = pool.work_list()
            if pool.P and (pl is None or nl > 0):
                self._call(self.lib.mlamr_flag_cells, pool.struct(), pool.state.data_ptr(), self.prm,
                           self._eta_rest.data_ptr(), self._wave_tol.data_ptr(), b["bits"].data_ptr(),
                           pool.blocks_per_patch(pool.max_interior), pl, nl, self.sh)
            self._reduce_flag_bits(b["bits"])
            self._call(self.lib.mlamr_flags_reference, b["bits"].data_ptr(), s.ny, s.nx, self.M,
                       self.pb.buffer_width, b["flags"].data_ptr(), b["allowed"].data_ptr(),
                       b["scratch"].data_ptr(), self.sh)
            region = self._region_mask_d(level)
            if region is not None:   # configured allowed rectangles (regrid.py:197-209)
                b["flags"].mul_(region)
                b["allowed"].mul_(region)
        return b["flags"], b["allowed"]

    def _region_mask_d(self, level: int):
        if not self.pb.allowed_regions:
            return None
        key = ("region", level)
        if key not in self._flagbuf:
            m = self.pb.region_mask(level).astype(np.uint8).reshape(-1)
            self._flagbuf[key] = arena().upload(m, self.dev, self.stream)
        return self._flagbuf[key]

    def _reduce_flag_bits(self, bits) -> None:
        """Single GPU: nothing to combine (the sharded driver all-reduces)."""

    def _cluster_level(self, level: int) -> np.ndarray:
        """Coarse boxes of the new finer level (cluster_flags, regrid.py:261)."""
        s = self.spec(level)
        if self._device_rule():
            flags_d, allowed_d = self._device_flags(level)
            cb = cluster_boxes_device(flags_d, allowed_d, s.ny, s.nx, self.pb.efficiency_target, self.stream)
            arena().reset()
            self.d2h_bytes += 8 * (s.ny + 1) * (s.nx + 1)
            return cb
        flags, allowed = self.flags_and_allowed(level)
        return cluster_boxes(flags, self.pb.efficiency_target, allowed)

    @staticmethod
    def _lexsorted(b: np.ndarray) -> np.ndarray:
        return b[np.lexsort((b[:, 0], b[:, 1]))] if len(b) else b

    def _rebuild(self, level: int, init: bool = False) -> bool:
        s = self.spec(level)
        rx, ry = s.r_x, s.r_y
        par = self.levels[level]
        old = self.levels.get(level + 1)
        fixed = self.pb.fixed_layout(level + 1) if init else None
        if fixed is not None:
            fb = np.asarray(fixed, dtype=np.int64).reshape(-1, 4)
            cb = np.stack([fb[:, 0] // rx, fb[:, 1] // ry, (fb[:, 2] + 1) // rx - 1, (fb[:, 3] + 1) // ry - 1], 1)
            cb = self._lexsorted(cb)
        else:
            with self._timed("regrid.flags+cluster"):
                cb = self._cluster_level(level)
            if self.pb.max_patch is not None:
                cb = chop_boxes(cb, *self.pb.max_patch, aligned=self.pb.chop_aligned)
        cb = np.asarray(cb, dtype=np.int64).reshape(-1, 4)
        nboxes = np.stack([cb[:, 0] * rx, cb[:, 1] * ry, (cb[:, 2] + 1) * rx - 1, (cb[:, 3] + 1) * ry - 1], 1)
        if old is not None:
            # the reference keeps the old patches when the sorted box lists
            # agree (regrid.py:265-268); an unchanged flag map gives the very
            # same list (clustering is deterministic), so the direct
            # comparison answers the common case without the sorts
            if np.array_equal(old.boxes, nboxes) or (
                    len(old.boxes) == len(nboxes)
                    and np.array_equal(self._lexsorted(old.boxes), self._lexsorted(nboxes))):
                return False
        elif len(nboxes) == 0:
            return False
        from .device import ALLOC_STATS
        f0 = ALLOC_STATS["fresh"]
        t0p = time.perf_counter()
        new = self._new_pool(level + 1, nboxes)
        self.host_prof["regrid.pool(fresh alloc)" if ALLOC_STATS["fresh"] > f0 else "regrid.pool(reuse)"] += \
            time.perf_counter() - t0p
        new.time = par.time
        M = self.M
        tq = time.perf_counter()
        with torch.cuda.stream(self.stream):
            if init and fixed is None and self.pb.init_mode == "scenario":
                self._set_initial(new)
            elif new.P:
                bpp = new.blocks_per_patch(new.max_interior // 4)   # copy pass: ~4 fine cells per thread
                part = self._scratch("refine", new.P * bpp * M)
                fs = self.spec(level + 1)
                ol = old.struct() if old is not None else empty_level_struct(fs, M)
                pl, nl = new.work_list()
                e0 = self._kt0()
                self._call(self.lib.mlamr_regrid_fill, new.struct(), ol, par.struct(), rx, ry, self.prm,
                           part.data_ptr(), bpp, self.status.data_ptr(), pl, nl, self.sh)
                if e0 is not None:
                    ob = old.boxes if old is not None else np.zeros((0, 4), np.int64)
                    self._kt1(f"k_regrid_fill L{level + 1}", e0,
                              lambda nb=nboxes, ob=ob: regrid_fill_bytes(nb, ob, rx, ry, M))
                if not init:
                    self._add_delta(0, part, new.P * bpp)
            new_child = paint_child_map(s, nboxes, rx, ry, self.dev, self.stream)
            if old is not None and old.P and not init:
                bpp = old.blocks_per_patch(old.max_interior // (rx * ry))
                part = self._scratch("derefine", old.P * bpp * M)
                pl, nl = old.work_list()
                self._call(self.lib.mlamr_derefine_delta, old.struct(), par.struct(), new_child.data_ptr(),
                           rx, ry, self.prm, part.data_ptr(), bpp, pl, nl, self.sh)
                self._add_delta(1, part, old.P * bpp)
        self.host_prof["regrid.fill+derefine"] += time.perf_counter() - tq
        tq = time.perf_counter()
        new.ghosts_in_cur = False
        self.levels[level + 1] = new
        if old is not None:
            old.release()
        if par.child is not None:
            release(par.child)
        par.child = new_child
        if level + 2 in self.levels:
            fs = self.spec(level + 1)
            if old is not None and old.child is not None:
                release(old.child)
            new.child = paint_child_map(fs, self.levels[level + 2].boxes, fs.r_x, fs.r_y, self.dev, self.stream)
        if not init:
            self.stats.num_regrids += 1
        self.host_prof["regrid.swap"] += time.perf_counter() - tq
        return True

    def regrid_from(self, level: int) -> None:
        t0 = time.perf_counter()
        if self._rebuild(level):
            for deeper in range(level + 1, self.L):
                self._rebuild(deeper)
        self.host_prof["regrid(total)"] += time.perf_counter() - t0

    # -- stepping (driver.py:224-309) ------------------------------------------------
    def _step_patches(self, level: int, dt: float, fused_siblings: bool = False, split=None) -> None:
        """``split`` = (n_first, between): step the first n_first tiles of the
        level's tile list, call ``between()`` (which may enqueue work and
        stream waits), then step the rest; one finalize over all tiles."""
        pool = self.levels[level]
        if pool.P == 0:
            return
        y_first = int(self.steps[level] % 2)
        # speed_bits are at "all dry" (-1) here: set at pool creation, and
        # reset by the previous finalize (reset_speeds) or level_speed
        src, dst = pool.state, pool.other
        lv = pool.struct(src)
        if _LOG_STEP_BYTES:
            b = pool.boxes if pool.owned is None else pool.boxes[pool.owned]
            nx, ny = b[:, 2] - b[:, 0] + 1, b[:, 3] - b[:, 1] + 1
            byts = int((8 * ((3 * self.M + 1) * (nx + 2) * (ny + 2) + 3 * self.M * nx * ny)).sum())
            import sys
            print(f"[mlamr] step level={level} tiles={pool.n_tiles} algorithmic_bytes={byts}", file=sys.stderr)
        timed = self.step_timer_level == level
        if timed:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
        gb = gp = None
        if fused_siblings:
            gbase, plan = pool.ghost_plan()[:2]
            gb, gp = gbase.data_ptr(), plan.data_ptr()
        if split is None:
            parts = [(0, pool.n_tiles)]
        else:
            parts = [(0, split[0]), (split[0], pool.n_tiles)]
        for k, (a, b) in enumerate(parts):
            if k == 1:
                split[1]()
            if b <= a:
                continue
            self._call(self.lib.mlamr_step, lv, src.data_ptr(), dst.data_ptr(), pool.tiles_d.data_ptr() + 12 * a,
                       b - a, pool.tile_tx, dt, y_first, self.prm, pool.speed_bits.data_ptr(),
                       pool.tile_acc.data_ptr() + 8 * (self.M + 2) * a, self.status.data_ptr(), gb, gp, self.sh)
        if timed:
            e1.record(self.stream)
            self.step_events.append((e0, e1, pool))
        self._call(self.lib.mlamr_step_finalize, lv, src.data_ptr(), dst.data_ptr(), pool.tiles_d.data_ptr(),
                   pool.n_tiles, dt, self.prm, pool.speed_bits.data_ptr(), pool.tile_acc.data_ptr(),
                   self.acc.data_ptr(), self.status.data_ptr(), self.bad.data_ptr(), int(not self.keep_step_speeds),
                   self.sh)
        pool.cur = 1 - pool.cur
        pool.ghosts_in_cur = False
        self.stats.total_cell_updates += pool.ncells
        self.stats.cell_updates_per_level[level] = self.stats.cell_updates_per_level.get(level, 0) + pool.ncells

    def _average_down(self, level: int) -> None:
        fine = self.levels.get(level + 1)
        coarse = self.levels[level]
        if fine is None or fine.P == 0 or coarse.P == 0:
            return
        if abs(fine.time - coarse.time) > _TIME_RTOL * max(1.0, abs(coarse.time)):
            raise TimeSyncError(f"level {level + 1} at t={fine.time!r} vs level {level} at t={coarse.time!r}")
        s = self.spec(level)
        cbase, n_coarse = fine.coarse_base(s.r_x, s.r_y)
        e0 = self._kt0()
        self._call(self.lib.mlamr_average_down_flat, fine.struct(), coarse.struct(), s.r_x, s.r_y, self.prm,
                   cbase.data_ptr(), n_coarse, self.status.data_ptr(), self.sh)
        # K4: per covered coarse cell 3M fine blocks read, 3M coarse written
        self._kt1(f"k_average_down L{level + 1}->L{level}", e0, 8 * 3 * self.M * (s.r_x * s.r_y + 1) * n_coarse)

    def advance_level(self, level: int, dt: float, t0: float) -> None:
        if level < self.L and self.steps[level] % self.pb.regrid_interval == 0:
            self.regrid_from(level)
        pool = self.levels[level]
        child = self.levels.get(level + 1)
        has_child = child is not None and child.P > 0
        # a level without children needs its ghost frames only for its own
        # step: the sibling part of the fill is fused into the step
        fuse = self.fuse_sibling_fill and not has_child
        self.fill_level_ghosts(level, t0, siblings=not fuse)
        self.levels[level].fused_frame = fuse   # the finite check reads its sibling cells via the plan
        self._step_patches(level, dt, fused_siblings=fuse)
        self.steps[level] += 1
        t1 = t0 + dt
        pool.time = t1
        if has_child:
            self.fill_level_ghosts(level, t1)
            self._stash[level] = (t0, dt, pool.other)
            s = self.spec(level)
            dtf = dt / s.r_t
            for k in range(s.r_t):
                self.advance_level(level + 1, dtf, t0 + k * dtf)
            self.levels[level + 1].time = t1
            self._average_down(level)
            del self._stash[level]

    # -- coarse step (driver.py:299-362) ----------------------------------------------
    def _speed_key(self, level: int):
        pool = self.levels.get(level)
        return (id(pool), pool.cur if pool is not None else -1, int(self.steps[level]), self._restores)

    def _enqueue_speed(self, pool) -> torch.Tensor:
        """k_max_speed over a level and the copy of its per-patch speed bits
        to pinned memory (read after the next synchronisation)."""
        self._call(self.lib.mlamr_max_speed_tiles, pool.struct(), pool.state.data_ptr(), pool.tiles_d.data_ptr(),
                   pool.n_tiles, pool.tile_tx, self.prm, pool.speed_bits.data_ptr(), self.sh)
        with torch.cuda.stream(self.stream):
            bits_h = self._pinned("speed", pool.P, torch.int64)
            bits_h.copy_(pool.speed_bits[:pool.P], non_blocking=True)
            dmemset(pool.speed_bits, 0xFF, self.stream)   # back to "all dry" (-1) for the next step
        return bits_h

    def level_speed(self, level: int) -> float:
        pool = self.levels.get(level)
        if pool is None or pool.P == 0:
            return 0.0
        cache = self._speed_cache
        if level == 1 and cache is not None and cache[0] == self._speed_key(1):
            bits = cache[1]   # read back with the previous step's mass
        else:
            bits_h = self._enqueue_speed(pool)
            self.stream.synchronize()
            self.d2h_bytes += 8 * pool.P
            bits = bits_h.numpy()
        sp = np.where(bits < 0, 0, bits).view(np.float64)
        return sp

    def choose_dt(self) -> float:
        """min over level-1 patches of physics.stable_dt (driver.py:337-339)."""
        dt = self.pb.dt_max
        with self._timed("dt"):
            sp = self.level_speed(1)
        s = self.spec(1)
        for v in sp:
            v = float(v)
            d = self.pb.dt_max if v <= 0.0 else min(self.pb.dt_max, self.pb.cfl * min(s.dx, s.dy) / v)
            dt = min(dt, d)
        return dt

    def apply_dynamic_rt(self, dt: float) -> None:
        if not self.pb.dynamic_rt:
            return
        dtl = dt
        for lev in range(1, self.L):
            s = self.spec(lev)
            fs = self.spec(lev + 1)
            sp = np.atleast_1d(np.asarray(self.level_speed(lev + 1), dtype=np.float64))
            # the running Python max from 0.0 skips NaN speeds (a NaN never
            # compares greater): the maximum of the non-NaN ones, floored at 0
            ok = sp[~np.isnan(sp)]
            vmax = max(0.0, float(ok.max())) if ok.size else 0.0
            rt = self.pb.pick_rt(vmax, dtl, min(fs.dx, fs.dy), max(s.r_x, s.r_y))
            self.specs[lev - 1] = replace(s, r_t=rt)
            dtl = dtl / rt

    def _add_delta(self, k: int, part: torch.Tensor, rows: int) -> None:
        """delta_acc[k] (0 refine, 1 derefine) and this coarse step's event
        delta (delta_acc[2]) += the column sums of a kernel's partials."""
        self._call(self.lib.mlamr_sum_partials, part.data_ptr(), rows, self.M, 1.0, self.delta_acc[k].data_ptr(),
                   self.delta_acc[2].data_ptr(), 0, self.sh)

    def advance_coarse_step(self, dt: float) -> None:
        self._call(self.lib.mlamr_sum_partials, None, 0, self.M, 1.0, self.delta_acc[2].data_ptr(), None, 1,
                   self.sh)
        with self._timed("advance(host enqueue)"):
            self.advance_level(1, dt, self.time)
        self.time += dt
        where = f"at t={self.time:.6g}"
        with self._timed("sync+mass+finite"):
            mass, event, nonfinite = self._step_readback(where)
        sync = mass - self._mass_prev - event
        if not self.stats.sync_delta:
            self.stats.sync_delta = [0.0] * self.M
        for m in range(self.M):
            self.stats.sync_delta[m] += float(sync[m])
        self._mass_prev = mass
        self.stats.num_coarse_steps += 1
        if nonfinite:
            # the reference counts the step, then checks finiteness (driver.py:299-309)
            raise_status(N.ST_NONFINITE, where)

    def _step_readback(self, where: str):
        """End of a coarse step with ONE host synchronisation: the composite
        mass and finite check (driver.py:286-297), this step's event delta,
        the status word, and -- for the next choose_dt -- level 1's observed
        speeds are enqueued and copied to pinned memory together; then the
        status is raised as the reference would: the advance's own errors
        here, a non-finite state (returned as a flag) by the caller after
        the step is counted."""
        M = self.M
        pool1 = self.levels.get(1)
        pre = pool1 is not None and pool1.P > 0
        with torch.cuda.stream(self.stream):
            tot = self._mass_device()
            self._reduce_event(self.delta_acc[2])
            hb = self._pinned("readback", 2 * M, torch.float64)
            hb[:M].copy_(tot, non_blocking=True)
            hb[M:].copy_(self.delta_acc[2], non_blocking=True)
            hs = self._pinned("status", 2, torch.int32)
            hs[:1].copy_(self.status, non_blocking=True)
            hs[1:].copy_(self.bad, non_blocking=True)
            if pre:
                bits_h = self._enqueue_speed(pool1)
        self.stream.synchronize()
        arena().reset()
        self.d2h_bytes += 16 * M + 8
        st = int(hs[0])
        nonfinite = bool(st & N.ST_NONFINITE)
        st &= ~N.ST_NONFINITE
        if st:
            self._speed_cache = None
            if st & N.ST_CFL:
                raise CflViolationError(f"Courant number > 1 on patch {int(hs[1])} {where}")
            raise_status(st, where)
        if pre and not nonfinite:
            self.d2h_bytes += 8 * pool1.P
            self._speed_cache = (self._speed_key(1), bits_h.numpy().copy())
        return hb[:M].numpy().copy(), hb[M:].numpy().copy(), nonfinite

    def _reduce_event(self, ev: torch.Tensor) -> None:
        """Single GPU: the refine/derefine delta of this coarse step is
        already global (the sharded driver all-reduces it, since mass is)."""

    def run(self, n_coarse: int) -> RunStats:
        for _ in range(n_coarse):
            dt = self.choose_dt()
            self.apply_dynamic_rt(dt)
            self.advance_coarse_step(dt)
        return self.finish()

    def run_until(self, t_final: float, frame_times=(), frame_callback=None) -> RunStats:
        """The reference's time loop (driver.py:312-362): level-1 stable dt,
        clipped to land exactly on the next frame time or t_final, with
        ``frame_callback(sim, time, index)`` at every due frame time.  Wall
        and CPU timers cover the integration loop only."""
        eps = 1e-12 * max(1.0, t_final)
        times = list(frame_times)
        idx = 0

        def emit():
            nonlocal idx
            while idx < len(times) and times[idx] <= self.time + eps:
                if frame_callback is not None:
                    frame_callback(self, self.time, idx)
                idx += 1

        emit()
        while self.time < t_final - eps:
            wall0, cpu0 = time.perf_counter(), time.process_time()
            dt = self.choose_dt()
            target = t_final if idx >= len(times) else min(t_final, times[idx])
            clipped = self.time + dt >= target - eps
            if clipped:
                dt = target - self.time
            self.apply_dynamic_rt(dt)
            self.advance_coarse_step(dt)
            if clipped:
                self.time = target
            self.stats.wall_time += time.perf_counter() - wall0
            self.stats.cpu_time += time.process_time() - cpu0
            emit()
        return self.finish()

    def finish(self) -> RunStats:
        """RunStats with the device accumulators folded in (idempotent: the
        fields are recomputed from the accumulators on every call)."""
        self.stream.synchronize()
        return self._fill_stats(self.stats, self.acc.cpu().numpy(), self.delta_acc.cpu().numpy())

    def _fill_stats(self, st: RunStats, acc: np.ndarray, d: np.ndarray) -> RunStats:
        M = self.M
        st.clipped_mass = list(acc[:M])
        st.hyperbolicity_warnings = int(round(acc[M]))
        st.wet_prefix_repairs = int(round(acc[M + 1]))
        st.refine_delta = list(d[0])
        st.derefine_delta = list(d[1])
        st.final_mass = list(self._mass_prev)
        if st.initial_mass:
            st.mass_drift = [f - i for f, i in zip(st.final_mass, st.initial_mass)]
        return st

    # -- checkpoint: host snapshot / restore (pinned host buffers) ----------------------------
    def _interior_base(self, pool: LevelPool):
        """(device prefix sums of the patches' interior sizes, total)."""
        b = pool.boxes
        n = (b[:, 2] - b[:, 0] + 1) * (b[:, 3] - b[:, 1] + 1) if pool.P else np.zeros(0, np.int64)
        base = np.concatenate([[0], np.cumsum(n)[:-1]]).astype(np.int64) if pool.P else np.zeros(1, np.int64)
        return arena().upload(base, self.dev, self.stream), int(n.sum()) if pool.P else 0

    def snapshot(self, bathymetry: bool = False) -> dict:
        """Copy the hierarchy (the patches' interiors, layouts, clocks and
        counters) into pinned host memory.  Ghost frames are refilled before
        anything reads them, so only interiors are packed
        (mlamr_pack_interiors).  The pools' bathymetry is problem data every
        pool derives on the device from the problem's level arrays
        (mlamr_fill_bathymetry), so it is copied only with
        ``bathymetry=True``; a restore re-derives it otherwise."""
        snap = {"time": self.time, "steps": dict(self.steps), "specs": list(self.specs), "levels": {},
                "acc": None, "delta_acc": None, "mass_prev": np.array(self._mass_prev),
                "stats": copy.deepcopy(self.stats)}
        nbytes = 0
        with torch.cuda.stream(self.stream):
            from .device import pinned_acquire
            for lev, pool in self.levels.items():
                pbase, ntot = self._interior_base(pool)
                n3 = 3 * self.M * max(ntot, 1)
                packed = acquire(n3, torch.float64, self.dev, self.stream)
                self._call(self.lib.mlamr_pack_interiors, pool.struct(), pool.state.data_ptr(), packed.data_ptr(),
                           pbase.data_ptr(), max(ntot, 1), pool.max_interior, 0, self.sh)
                st = pinned_acquire(n3, torch.float64)
                st.copy_(packed, non_blocking=True)
                release(packed)
                ba = None
                if bathymetry:
                    ba = pinned_acquire(pool.bathy.numel(), torch.float64).view(pool.bathy.shape)
                    ba.copy_(pool.bathy, non_blocking=True)
                nbytes += st.numel() * 8 + (ba.numel() * 8 if ba is not None else 0)
                # interiors only: a restored pool's frames are refilled first
                snap["levels"][lev] = {"boxes": pool.boxes.copy(), "state": st, "bathy": ba, "time": pool.time,
                                       "ghosts": False}
            acc = torch.empty(self.acc.shape, dtype=torch.float64, pin_memory=True)
            acc.copy_(self.acc, non_blocking=True)
            dacc = torch.empty(self.delta_acc.shape, dtype=torch.float64, pin_memory=True)
            dacc.copy_(self.delta_acc, non_blocking=True)
        self.stream.synchronize()
        snap["acc"], snap["delta_acc"] = acc, dacc
        snap["nbytes"] = nbytes
        self.d2h_bytes += nbytes
        return snap

    def close(self) -> None:
        """Hand every level pool's buffers to the recycle list (device.release)
        so a simulation built next -- e.g. a restore from this one's
        snapshot -- reuses them instead of calling cudaMalloc.  The
        simulation is unusable afterwards."""
        for pool in self.levels.values():
            pool.release()
        self.levels = {}

    @staticmethod
    def release_snapshot(snap: dict) -> None:
        """Hand a snapshot's pinned buffers back for reuse by later
        snapshots (after any restore from it has been issued: reuse is
        ordered on the driver stream)."""
        from .device import pinned_release
        for d in snap.get("levels", {}).values():
            for key in ("state", "bathy"):
                if d.get(key) is not None:
                    pinned_release(d[key])
                    d[key] = None

    @classmethod
    def restore(cls, problem, snap: dict, device: str = "cuda", stream=None,
                reserve_factor: float = 0.0) -> "Simulation":
        """Rebuild a device hierarchy from :meth:`snapshot` output (host->device)."""
        return cls(problem, device=device, stream=stream, _restore=snap, reserve_factor=reserve_factor)

    def _restore_pool(self, lev: int, d: dict) -> LevelPool:
        """An empty pool for a level of a snapshot (sharded runs add ownership)."""
        return LevelPool(self.spec(lev), d["boxes"], self.M, self.dev, self.stream, need_gown=lev < self.L)

    def _level_boxes(self, lev: int) -> np.ndarray:
        """All boxes of a level (a sharded run's pools hold only some)."""
        return self.levels[lev].boxes

    def _restore_from(self, snap: dict) -> None:
        self._speed_cache = None
        self._restores += 1
        self.time = snap["time"]
        self.steps = dict(snap["steps"])
        self.specs = list(snap["specs"])
        self.stats = copy.deepcopy(snap["stats"])
        nbytes = 0
        for lev in sorted(snap["levels"]):
            d = snap["levels"][lev]
            pool = self._restore_pool(lev, d)
            with torch.cuda.stream(self.stream):
                pbase, ntot = self._interior_base(pool)
                packed = acquire(d["state"].numel(), torch.float64, self.dev, self.stream)
                packed.copy_(d["state"], non_blocking=True)
                self._call(self.lib.mlamr_pack_interiors, pool.struct(), pool.state.data_ptr(), packed.data_ptr(),
                           pbase.data_ptr(), max(ntot, 1), pool.max_interior, 1, self.sh)
                release(packed)
                if d["bathy"] is not None:
                    pool.bathy.copy_(d["bathy"], non_blocking=True)
            if d["bathy"] is None and pool.P:
                self._call(self.lib.mlamr_fill_bathymetry, pool.struct(), self.level_bathy[lev - 1].data_ptr(),
                           self.bcs, self.sh)
            nbytes += d["state"].numel() * 8 + (d["bathy"].numel() * 8 if d["bathy"] is not None else 0)
            pool.time = d["time"]
            pool.ghosts_in_cur = d["ghosts"]
            self.levels[lev] = pool
        for lev in range(1, self.L):
            if lev + 1 in self.levels:
                s = self.spec(lev)
                self.levels[lev].child = paint_child_map(s, self._level_boxes(lev + 1), s.r_x, s.r_y,
                                                         self.dev, self.stream)
        with torch.cuda.stream(self.stream):
            self.acc.copy_(snap["acc"], non_blocking=True)
            self.delta_acc.copy_(snap["delta_acc"], non_blocking=True)
        self._mass_prev = np.array(snap["mass_prev"])
        self.h2d_bytes += nbytes

    # -- host views (tests, frames) ------------------------------------------------------
    def patch_fields(self, level: int):
        """List of (box, h, hu, hv, bathy) host arrays for every patch of a level."""
        pool = self.levels[level]
        host = pool.download()
        out = []
        for p in range(pool.P):
            h, hu, hv, b = pool.patch_arrays(p, host=host)
            out.append((tuple(int(v) for v in pool.boxes[p]), h, hu, hv, b))
        return out


def run_simulation(problem, out_dir=None, t_final: float | None = None, frame_times=(), text_frames: bool = False,
                   n_coarse: int | None = None, sim_cls=None, **kw) -> RunStats:
    """``run_simulation`` of the reference (driver.py:365-410): run, write
    ``frameNNNN.bin|txt`` at the frame times and ``stats.json`` into
    ``out_dir``; on a numerical abort or CFL violation write ``abort.*``
    and the partial stats before re-raising.  Frames come straight from the
    device pools (frames.py).  ``n_coarse`` runs a fixed number of coarse
    steps instead of a time span (frames at t=0 and at the end)."""
    from pathlib import Path
    from . import frames as F
    sim = (sim_cls or Simulation)(problem, **kw)
    sim.stats.amr_enabled = bool(getattr(problem, "amr_enabled", len(problem.ratios_x) > 0))
    out = Path(out_dir) if out_dir is not None else None
    if out is not None and getattr(sim, "rank", 0) == 0:
        out.mkdir(parents=True, exist_ok=True)
    ext = "txt" if text_frames else "bin"

    def frame_cb(s, t, index):
        if out is not None:
            F.write_frame(s, out / f"frame{index:04d}.{ext}", text_frames)

    try:
        if n_coarse is not None:
            frame_cb(sim, sim.time, 0)
            stats = sim.run(n_coarse)
            frame_cb(sim, sim.time, 1)
        else:
            stats = sim.run_until(t_final, frame_times, frame_cb)
    except (NumericalAbortError, CflViolationError):
        if out is not None:
            F.write_frame(sim, out / f"abort.{ext}", text_frames)
            if getattr(sim, "rank", 0) == 0:
                sim.stats.to_json(out / "stats.json")
        raise
    if out is not None and getattr(sim, "rank", 0) == 0:
        stats.to_json(out / "stats.json")
    return stats
