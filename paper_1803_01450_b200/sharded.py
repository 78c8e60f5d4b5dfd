"""Multi-GPU driver: the subcycled recursion of :class:`driver.Simulation`
over SFC-sharded patch ownership with shadow replicas (distributed.py).

Differences from the single-GPU driver, all confined to this subclass:

* every level keeps its global layout and owner array; the local pool
  holds owned + shadow patches in global list order, so the owner maps'
  precedence equals the reference's list order (ghost.py:58-84);
* stepping, filling, flagging and reductions run over owned patches only
  (patch lists / owned tiles); coarsening runs over every local fine
  patch into the local coarse pool, and the coarse owner's result counts;
* shadows are refreshed by whole-patch transfers from their owners
  (i) at the start of a level's advance, (ii) after its t0 ghost fill
  (their frames then sit in the buffer that becomes the stash),
  (iii) after its t1 fill, and (iv) for the finer level before it is
  averaged down;
* a regrid all-reduces the flag bits, clusters identically on every rank,
  partitions the new layout along the Morton curve and reshapes the
  affected pools (parents of old and new owned patches, old patches
  overlapping new owned ones, children needed by new coarse owners);
* dt / dynamic-r_t speeds are all-reduced maxima, composite mass and
  counters all-reduced sums, the status word an all-reduced maximum.
"""

from __future__ import annotations

import copy
from math import prod

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N
from .device import LevelPool, dmemset, empty_level_struct, paint_child_map
from .distributed import (Comm, Transfer, _any_meet, needed, partition, patch_sizes, plan_acquire, plan_refresh,
                          ring_segments, run_transfer)
from .driver import Simulation
from .mesh import GHOST_WIDTH, IndexBox, boxes_array
from .regrid import chop_boxes, cluster_boxes

_EMPTY = np.zeros((0, 4), np.int64)


class ShardedSimulation(Simulation):
    def __init__(self, problem, comm: Comm | None = None, device: str = "cuda", stream=None,
                 reserve_factor: float = 2.0, _restore: dict | None = None):
        self._init_sharding(comm)
        self._common_init(problem, device, stream)
        self._xstream = torch.cuda.Stream(device=self.dev)
        with torch.cuda.stream(self.stream):
            self.comm.warmup_p2p(self.dev)
        if _restore is not None:
            self._restore_from(_restore)
            return
        # level 1 as aligned tiles spread over the ranks like any other
        # level (bit-identical to the reference's single level-1 patch:
        # Simulation.level1_boxes); 128-cell tiles unless MLAMR_L1_TILE says
        # otherwise (C4's 512^2 level 1: 16 tiles), one patch if the domain
        # fits one tile or the job has one rank
        b1 = self.level1_boxes(128 if self.world > 1 else 0)
        layouts, owners = {1: b1}, {1: partition(b1, *self._scale(1), self.world)}
        self.layout[1] = b1
        self.owner[1] = owners[1]
        self.held[1] = self._held_all(1, layouts, owners)
        self.full[1] = self._full_all(1, layouts, owners)
        base = self._make_pool(1, b1, self.owner[1], self.held[1][self.rank])
        self._set_initial(base)
        self.levels[1] = base
        for lev in range(1, self.L):
            self._rebuild(lev, init=True)
        self._mass_prev = self.composite_mass()
        self.stats.initial_mass = list(self._mass_prev)
        if reserve_factor > 0:
            from .device import reserve
            reserve(int(reserve_factor * self.device_bytes()), self.dev, self.stream)

    def _init_sharding(self, comm) -> None:
        self.comm = comm or Comm()
        self.rank, self.world = self.comm.rank, self.comm.world
        self.layout, self.owner, self.held = {}, {}, {}
        # per level and rank: the held patches needed in full (owned, parents,
        # children); the other shadows are refreshed as interior rings
        self.full = {}
        self.ring_refresh = True
        self._xstream = None   # the shadow-exchange stream (set with the device)
        # (ii) on the exchange stream, overlapping the step.  Off by default:
        # with NCCL it puts point-to-point traffic on a second stream next to
        # the driver stream's collectives, which this build could not run
        # (one GPU; NCCL refuses two ranks on one device).  The gloo tests
        # exercise it (tests/test_gpu_sharded.py sets MLAMR_OVERLAP_REFRESH).
        import os as _os
        self.overlap_refresh = _os.environ.get("MLAMR_OVERLAP_REFRESH", "0") == "1"
        self._ring_cache = {}
        self._fullc_cache = {}
        self.bytes_exchanged = 0

    # -- checkpoint: per-rank snapshot of its pools (owned + shadows) -------------
    def snapshot(self) -> dict:
        """This rank's part of the hierarchy (Simulation.snapshot of its pools)
        plus the global layouts and ownership, for restore() by the same
        rank of a job of the same size."""
        snap = super().snapshot()
        cp = lambda d: {k: {r: a.copy() for r, a in v.items()} for k, v in d.items()}
        snap["sharded"] = {
            "world": self.world, "rank": self.rank,
            "layout": {k: v.copy() for k, v in self.layout.items()},
            "owner": {k: v.copy() for k, v in self.owner.items()},
            "held": cp(self.held), "full": cp(self.full),
            "local": {lev: (pool.gidx.copy(), None if pool.owned is None else pool.owned.copy())
                      for lev, pool in self.levels.items()},
        }
        return snap

    @classmethod
    def restore(cls, problem, snap: dict, comm: Comm | None = None, device: str = "cuda",
                stream=None) -> "ShardedSimulation":
        return cls(problem, comm=comm, device=device, stream=stream, _restore=snap)

    def _restore_from(self, snap: dict) -> None:
        sh = snap["sharded"]
        if sh["world"] != self.world or sh["rank"] != self.rank:
            raise ValueError(f"snapshot of rank {sh['rank']}/{sh['world']} restored on rank {self.rank}/{self.world}")
        self.layout = {k: v.copy() for k, v in sh["layout"].items()}
        self.owner = {k: v.copy() for k, v in sh["owner"].items()}
        self.held = {k: {r: a.copy() for r, a in v.items()} for k, v in sh["held"].items()}
        self.full = {k: {r: a.copy() for r, a in v.items()} for k, v in sh["full"].items()}
        self._restore_local = sh["local"]
        super()._restore_from(snap)

    def _restore_pool(self, lev: int, d: dict) -> LevelPool:
        gidx, owned = self._restore_local[lev]
        return LevelPool(self.spec(lev), d["boxes"], self.M, self.dev, self.stream, need_gown=lev < self.L,
                         owned=owned, gidx=gidx)

    def _level_boxes(self, lev: int) -> np.ndarray:
        return self.layout[lev]

    # -- geometry helpers -----------------------------------------------------
    def _scale(self, level: int):
        sx = prod(s.r_x for s in self.specs[level - 1:self.L - 1])
        sy = prod(s.r_y for s in self.specs[level - 1:self.L - 1])
        return sx, sy

    def _ratios(self):
        return {s.level: (s.r_x, s.r_y) for s in self.specs}

    def _held_all(self, level, layouts, owners, extra=None, full_only=False, with_children=True):
        R = self._ratios()
        return {r: needed(level, r, layouts, owners, R, None if extra is None else extra(r), full_only=full_only,
                          with_children=with_children)
                for r in range(self.world)}

    def _full_all(self, level, layouts, owners, extra=None):
        """Per rank: the held patches every refresh sends whole (owned and
        parents); children are sent whole only by the pre-coarsening refresh."""
        return self._held_all(level, layouts, owners, extra, full_only=True, with_children=False)

    def _full_coarsen(self, level: int):
        key = (level, id(self.layout.get(level)), id(self.layout.get(level - 1)))
        ent = self._fullc_cache.get(level)
        if ent is None or ent[0] != key:
            ent = (key, self._held_all(level, self.layout, self.owner, full_only=True, with_children=True))
            self._fullc_cache[level] = ent
        return ent[1]

    def _make_pool(self, level, gboxes, owner, local_g) -> LevelPool:
        local_g = np.asarray(local_g, np.int64)
        pool = LevelPool(self.spec(level), gboxes[local_g] if len(local_g) else _EMPTY, self.M, self.dev,
                         self.stream, need_gown=level < self.L, owned=owner[local_g] == self.rank,
                         gidx=local_g)
        if pool.P:
            self._call(self.lib.mlamr_fill_bathymetry, pool.struct(), self.level_bathy[level - 1].data_ptr(),
                       self.bcs, self.sh)
        return pool

    # -- shadow transfers --------------------------------------------------------
    def _ring_table(self, level):
        """CSR view of ring_segments() for the level's layout (cached)."""
        lay = self.layout[level]
        key = (level, id(lay), len(lay))
        ent = self._ring_cache.get(level)
        if ent is None or ent[0] != key:
            rp, ro, ln, rsize = ring_segments(lay)
            cnt = np.bincount(rp, minlength=len(lay)).astype(np.int64)
            start = np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(np.int64)
            ent = (key, ro, ln, rsize, cnt, start)
            self._ring_cache[level] = ent
        return ent[1:]

    def _transfer(self, level, tr, src: LevelPool, dst: LevelPool, stream=None) -> None:
        st = stream or self.stream
        full_sz = patch_sizes(self.layout[level])
        ro, ln, rsize, cnt, start = self._ring_table(level)
        M3 = 3 * self.M

        def nsz(g, ring):
            if ring is None:
                return full_sz[g]
            return np.where(ring, rsize[g], full_sz[g])

        def runs(g, ring, block_off):
            """(block-relative absolute offsets, packed offsets, lengths) of
            the runs that move for patches g whose blocks start at block_off."""
            sz = nsz(g, ring)
            poff = np.concatenate([[0], np.cumsum(sz)[:-1]]).astype(np.int64)
            if ring is None or not ring.any():
                return np.asarray(block_off, np.int64), poff, sz
            r = np.asarray(ring, bool)
            k = np.flatnonzero(r)
            c = cnt[g[k]]
            idx = np.repeat(start[g[k]], c) + (np.arange(int(c.sum())) - np.repeat(np.cumsum(c) - c, c))
            r_len = ln[idx]
            r_abs = np.repeat(np.asarray(block_off, np.int64)[k], c) + ro[idx]
            # packed offsets: each ring patch's runs are consecutive from its poff
            cum = np.cumsum(r_len) - r_len
            first = np.repeat(np.cumsum(c) - c, c)
            r_pack = np.repeat(poff[k], c) + (cum - cum[first])
            f = np.flatnonzero(~r)
            return (np.concatenate([np.asarray(block_off, np.int64)[f], r_abs]),
                    np.concatenate([poff[f], r_pack]), np.concatenate([full_sz[g[f]], r_len]))

        def pack(g, ring, src_off, buf):
            a, pk, lens = runs(g, ring, src_off)
            n = int(nsz(g, ring).sum())
            src.copy_segments(src.state, src.FS, buf, n, a, pk, lens, stream=st)

        def unpack(g, ring, buf, dst_off):
            a, pk, lens = runs(g, ring, dst_off)
            n = int(nsz(g, ring).sum())
            dst.copy_segments(buf, n, dst.state, dst.FS, pk, a, lens, stream=st)

        with torch.cuda.stream(st):
            self.bytes_exchanged += run_transfer(
                self.comm, tr, nsz, M3, lambda g: src.offsets[src.local_of(g)],
                lambda g: dst.offsets[dst.local_of(g)], pack, unpack, torch.float64, self.dev)

    def _refresh(self, level: int, coarsen: bool = False, full_only: bool = False, stream=None) -> None:
        """Shadow refresh; ``coarsen``: the one in front of averaging this
        level down, which must deliver children whole.  ``full_only``: only
        the shadows held in full (their frames were just filled; the
        ring-only ones have not changed since the last refresh)."""
        if self.world == 1 or level not in self.levels:
            return
        full = None
        if self.ring_refresh:
            full = self._full_coarsen(level) if coarsen else self.full.get(level)
        tr = plan_refresh(self.rank, self.world, self.held[level], self.owner[level], full)
        if full_only and tr.send_ring is not None:
            keep = lambda d, ring: {q: g[~ring[q]] for q, g in d.items() if (~ring[q]).any()}
            tr = Transfer(keep(tr.send, tr.send_ring), keep(tr.recv, tr.recv_ring),
                          {q: np.zeros(int((~r).sum()), bool) for q, r in tr.send_ring.items() if (~r).any()},
                          {q: np.zeros(int((~r).sum()), bool) for q, r in tr.recv_ring.items() if (~r).any()})
        pool = self.levels[level]
        self._transfer(level, tr, pool, pool, stream=stream)

    def _reshape(self, level: int, new_held, new_full=None) -> None:
        """Replace a level's local pool by one holding new_held[rank] (same
        layout and owners), moving data: local copies + owners' sends.
        Patches held only as refreshed rings are not complete, so they are
        fetched whole from their owners rather than copied locally.
        ``new_full`` = the patches each rank needs in full afterwards
        (default: all of new_held)."""
        if new_full is None:
            new_full = new_held
        old = self.levels[level]
        want = new_held[self.rank]
        # the skip must be a collective decision: a rank whose own set is
        # unchanged may still have to send patches to a rank whose set grew
        old_full = self.full.get(level, self.held[level])
        if all(np.array_equal(new_held[r], self.held[level][r]) and np.array_equal(new_full[r], old_full[r])
               for r in range(self.world)):
            self.held[level] = new_held
            self.full[level] = new_full
            return
        have = {r: (np.intersect1d(self.held[level][r], old_full[r], assume_unique=True)
                    if self.ring_refresh else self.held[level][r]) for r in range(self.world)}
        new = self._make_pool(level, self.layout[level], self.owner[level], want)
        common = np.intersect1d(have[self.rank], want, assume_unique=True)
        if len(common):
            sizes = patch_sizes(self.layout[level])[common]
            with torch.cuda.stream(self.stream):
                new.copy_segments(old.state, old.FS, new.state, new.FS, old.offsets[old.local_of(common)],
                                  new.offsets[new.local_of(common)], sizes)
        tr = plan_acquire(self.rank, self.world, have, new_held, self.owner[level])
        self._transfer(level, tr, old, new)
        new.time = old.time
        new.ghosts_in_cur = old.ghosts_in_cur
        new.child = old.child
        self.levels[level] = new
        self.held[level] = new_held
        self.full[level] = new_full
        old.release()

    # -- reductions ------------------------------------------------------------------
    def _sync_status(self, where: str = "") -> None:
        with torch.cuda.stream(self.stream):
            self.comm.allreduce(self.status, dist.ReduceOp.MAX if self.world > 1 else None)
            self.comm.allreduce(self.bad, dist.ReduceOp.MIN if self.world > 1 else None)
        super()._sync_status(where)

    def _step_readback(self, where: str):
        """Status, mass and event delta all-reduced over the ranks (the
        single-GPU readback batches them into one synchronisation)."""
        self._sync_status(where)
        mass = self.composite_mass()
        with torch.cuda.stream(self.stream):
            ev = self.delta_acc[2].clone()
            self._reduce_event(ev)
        self.stream.synchronize()
        self.d2h_bytes += 8 * self.M
        event = ev.cpu().numpy()
        with torch.cuda.stream(self.stream):
            self.comm.allreduce(self.status, dist.ReduceOp.MAX if self.world > 1 else None)
        self.stream.synchronize()
        nonfinite = bool(int(self.status.item()) & N.ST_NONFINITE)
        return mass, event, nonfinite

    def composite_mass(self) -> np.ndarray:
        with torch.cuda.stream(self.stream):
            tot = self._mass_device().clone()
            self.comm.allreduce(tot)
        self.stream.synchronize()
        from .device import arena
        arena().reset()
        return tot.cpu().numpy()

    def level_speed(self, level: int):
        pool = self.levels.get(level)
        with torch.cuda.stream(self.stream):
            best = torch.full((1,), -1, dtype=torch.int64, device=self.dev)
            if pool is not None and pool.P:
                dmemset(pool.speed_bits, 0xFF, self.stream)
                if pool.n_tiles:
                    self._call(self.lib.mlamr_max_speed_tiles, pool.struct(), pool.state.data_ptr(),
                               pool.tiles_d.data_ptr(), pool.n_tiles, pool.tile_tx, self.prm,
                               pool.speed_bits.data_ptr(),
                               self.sh)
                best = torch.max(pool.speed_bits[:pool.P]).reshape(1)
                dmemset(pool.speed_bits, 0xFF, self.stream)   # back to "all dry" for the next step (see the driver)
            self.comm.allreduce(best, dist.ReduceOp.MAX if self.world > 1 else None)
        self.stream.synchronize()
        b = int(best.item())
        # stable_dt is monotone in the speed, so the minimum over patches of
        # the per-patch dt equals dt of the global maximum speed (bit for bit)
        return np.array([0.0 if b < 0 else np.array([b], np.int64).view(np.float64)[0]])

    def finish(self):
        """Global RunStats of the job: the accumulators, total and per-level
        cell counts are all-reduced into temporaries and returned in a copy,
        so this rank's live accumulators and ``self.stats`` keep counting
        their own patches (finish() may be called any number of times)."""
        levels = [s.level for s in self.specs]
        with torch.cuda.stream(self.stream):
            acc = self.acc.clone()
            dacc = self.delta_acc.clone()
            self.comm.allreduce(acc)
            self.comm.allreduce(dacc)
            cells = torch.tensor([float(self.stats.total_cell_updates)]
                                 + [float(self.stats.cell_updates_per_level.get(l, 0)) for l in levels],
                                 dtype=torch.float64, device=self.dev)
            self.comm.allreduce(cells)
        self.stream.synchronize()
        st = self._fill_stats(copy.deepcopy(self.stats), acc.cpu().numpy(), dacc.cpu().numpy())
        c = [int(v) for v in cells.cpu().tolist()]
        st.total_cell_updates = c[0]
        st.cell_updates_per_level = {l: n for l, n in zip(levels, c[1:]) if n}
        return st

    def _reduce_event(self, ev: torch.Tensor) -> None:
        """The refine/derefine deltas accumulate over owned patches only,
        while the composite mass is global: the per-step event delta must be
        global too before sync = mass - mass_prev - event (driver.py:303-307)."""
        self.comm.allreduce(ev)

    # -- flags over owned patches, all-reduced -----------------------------------------
    def _reduce_flag_bits(self, bits) -> None:
        """Each rank wrote the bits of its owned cells only: max == union."""
        if self.world > 1:
            self.comm.allreduce(bits, dist.ReduceOp.MAX)   # uint8 in place

    def _device_rule(self) -> bool:
        # a rank's owner maps hold only its local patches: Bernoulli coverage
        # comes from the global layout on the host; the gradient rule runs
        # in two device halves around the union of the owned flags
        return self.pb.flag_rule[0] in ("reference", "gradient")

    def _device_flags(self, level: int):
        if self.pb.flag_rule[0] != "gradient":
            return super()._device_flags(level)
        from .device import arena
        from .mesh import paint
        pool = self.levels[level]
        s = self.spec(level)
        b = self._flag_buffers(level)
        _, tol, width, layers = self.pb.flag_rule
        mask = 0
        for m in layers:
            mask |= 1 << int(m)
        key = ("eta", level)
        with torch.cuda.stream(self.stream):
            if key not in self._flagbuf:
                self._flagbuf[key] = torch.empty(len(layers) * s.ny * s.nx, dtype=torch.float64, device=self.dev)
            n = s.ny * s.nx
            if pool.P:
                owned = arena().upload(np.asarray(pool.owned, np.uint8), self.dev, self.stream)
                self._call(self.lib.mlamr_flags_gradient_raw, pool.struct(), pool.state.data_ptr(), self.prm, mask,
                           float(tol), owned.data_ptr(), b["bits"].data_ptr(), b["scratch"].data_ptr(),
                           self._flagbuf[key].data_ptr(), self.sh)
            else:
                dmemset(b["bits"], 0, self.stream)
            self._reduce_flag_bits(b["bits"])          # union of the ranks' owned flags
            cov = arena().upload(paint(self.layout[level], s.ny, s.nx).astype(np.uint8).reshape(-1),
                                 self.dev, self.stream)
            self._call(self.lib.mlamr_flags_finish, b["bits"].data_ptr(), cov.data_ptr(), s.ny, s.nx, int(width),
                       b["flags"].data_ptr(), b["allowed"].data_ptr(), b["scratch"].data_ptr(), self.sh)
            region = self._region_mask_d(level)
            if region is not None:
                b["flags"].mul_(region)
                b["allowed"].mul_(region)
        return b["flags"], b["allowed"]

    def flags_and_allowed(self, level: int):
        s = self.spec(level)
        if self.pb.flag_rule[0] == "bernoulli":
            from .mesh import dilate, paint
            from .regrid import nesting_allowed
            covered = paint(self.layout[level], s.ny, s.nx)
            f = self.pb.bernoulli_flags(level, self.steps[level])
            f = dilate(f, self.pb.flag_rule[2]) & covered
            allowed = nesting_allowed(self.layout[level], s.ny, s.nx)
            region = self.pb.region_mask(level)
            if region is not None:
                allowed = allowed & region
            return f & allowed, allowed
        return super().flags_and_allowed(level)

    # -- regrid --------------------------------------------------------------------------
    def _rebuild(self, level: int, init: bool = False) -> bool:
        s = self.spec(level)
        rx, ry = s.r_x, s.r_y
        fixed = self.pb.fixed_layout(level + 1) if init else None
        if fixed is not None:
            fb = np.asarray(fixed, dtype=np.int64).reshape(-1, 4)
            cb = np.stack([fb[:, 0] // rx, fb[:, 1] // ry, (fb[:, 2] + 1) // rx - 1, (fb[:, 3] + 1) // ry - 1], 1)
            cb = self._lexsorted(cb)
        else:
            cb = self._cluster_level(level)
            if self.pb.max_patch is not None:
                cb = chop_boxes(cb, *self.pb.max_patch, aligned=self.pb.chop_aligned)
        cb = np.asarray(cb, dtype=np.int64).reshape(-1, 4)
        nboxes = np.stack([cb[:, 0] * rx, cb[:, 1] * ry, (cb[:, 2] + 1) * rx - 1, (cb[:, 3] + 1) * ry - 1], 1)
        old_layout = self.layout.get(level + 1, _EMPTY)
        old_owner = self.owner.get(level + 1, np.zeros(0, np.int32))
        if level + 1 in self.levels:
            if np.array_equal(old_layout, nboxes) or (
                    len(old_layout) == len(nboxes)
                    and np.array_equal(self._lexsorted(old_layout), self._lexsorted(nboxes))):
                return False
        elif len(nboxes) == 0:
            return False
        new_owner = partition(nboxes, *self._scale(level + 1), self.world)
        layouts = dict(self.layout)
        owners = dict(self.owner)
        layouts[level + 1] = nboxes
        owners[level + 1] = new_owner
        # (a) the parent level must hold the stencils of new and old owned fine patches
        ext_fine = lambda r: {level + 1: old_layout[old_owner == r]}  # noqa: E731
        self._reshape(level, self._held_all(level, layouts, owners, ext_fine),
                      self._full_all(level, layouts, owners, ext_fine))
        par = self.levels[level]
        # (b) old fine patches overlapping new owned patches
        old = self.levels.get(level + 1)
        if old is not None:
            ext = {}
            for r in range(self.world):
                hit = np.flatnonzero(_any_meet(old_layout, nboxes[new_owner == r]))
                ext[r] = np.union1d(self.held[level + 1][r], hit).astype(np.int64)
            self._reshape(level + 1, ext)
            old = self.levels[level + 1]
        # (c) the new level
        held_new = self._held_all(level + 1, layouts, owners)
        full_new = self._full_all(level + 1, layouts, owners)
        new = self._make_pool(level + 1, nboxes, new_owner, held_new[self.rank])
        new.time = par.time
        M = self.M
        with torch.cuda.stream(self.stream):
            if init and fixed is None and self.pb.init_mode == "scenario":
                self._set_initial(new)
            elif new.P:
                bpp = new.blocks_per_patch(new.max_interior // 4)   # copy pass: ~4 fine cells per thread
                part = self._scratch("refine", new.P * bpp * M)
                ol = old.struct() if old is not None else empty_level_struct(self.spec(level + 1), M)
                pl, nl = new.work_list()
                if nl > 0:
                    self._call(self.lib.mlamr_regrid_fill, new.struct(), ol, par.struct(), rx, ry, self.prm,
                               part.data_ptr(), bpp, self.status.data_ptr(), pl, nl, self.sh)
                if not init:
                    self._add_delta(0, part, new.P * bpp)
            new_child = paint_child_map(s, nboxes, rx, ry, self.dev, self.stream)
            if old is not None and old.P and not init:
                bpp = old.blocks_per_patch(old.max_interior // (rx * ry))
                part = self._scratch("derefine", old.P * bpp * M)
                pl, nl = old.work_list()
                if nl > 0:
                    self._call(self.lib.mlamr_derefine_delta, old.struct(), par.struct(), new_child.data_ptr(),
                               rx, ry, self.prm, part.data_ptr(), bpp, pl, nl, self.sh)
                self._add_delta(1, part, old.P * bpp)
        # (d) install and fill the new shadows from their owners
        self.layout[level + 1] = nboxes
        self.owner[level + 1] = new_owner
        self.held[level + 1] = held_new
        self.full[level + 1] = full_new
        self.levels[level + 1] = new
        if old is not None:
            old.release()
        par.child = new_child
        self._refresh(level + 1)
        # (e) the level below the new one: its shadow set depends on the new owners
        if level + 2 in self.levels:
            self._reshape(level + 2, self._held_all(level + 2, layouts, owners),
                          self._full_all(level + 2, layouts, owners))
            fs = self.spec(level + 1)
            new.child = paint_child_map(fs, self.layout[level + 2], fs.r_x, fs.r_y, self.dev, self.stream)
        if not init:
            self.stats.num_regrids += 1
        return True

    # -- recursion with refresh points -------------------------------------------------
    def _split_tiles(self, level: int) -> int:
        """Order the finest level's tiles so that those whose step reads no
        shadow (no halo cell inside a foreign sibling, patch not touching the
        level box, whose BC corners read copied cells) come first; returns
        their number (cached per pool and layout)."""
        pool = self.levels[level]
        key = (id(pool), pool.n_tiles)
        if getattr(pool, "_split_key", None) == key:
            return pool._n_indep
        tl = pool.tiles
        b = pool.boxes
        ty, tx = pool.tile_shape
        p = tl[:, 0]
        lo_i = b[p, 0] + tl[:, 2]
        lo_j = b[p, 1] + tl[:, 1]
        pad = np.stack([lo_i - 1, lo_j - 1, np.minimum(lo_i + tx - 1, b[p, 2]) + 1,
                        np.minimum(lo_j + ty - 1, b[p, 3]) + 1], axis=1)
        shadows = b[~pool.owned] if pool.owned is not None else _EMPTY
        dep = _any_meet(pad, shadows) if len(shadows) else np.zeros(len(tl), bool)
        s = self.spec(level)
        touch = (b[:, 0] == 0) | (b[:, 2] == s.nx - 1) | (b[:, 1] == 0) | (b[:, 3] == s.ny - 1)
        dep = dep | touch[p]
        pool.reorder_tiles(np.concatenate([np.flatnonzero(~dep), np.flatnonzero(dep)]))
        pool._split_key = (id(pool), pool.n_tiles)
        pool._n_indep = int((~dep).sum())
        return pool._n_indep

    def advance_level(self, level: int, dt: float, t0: float) -> None:
        if (self.overlap_refresh and self.world > 1 and level == self.L and self.fuse_sibling_fill
                and level in self.levels and self.levels[level].P):
            self._advance_finest_overlapped(level, dt, t0)
            return
        self._refresh(level)                                            # (i)
        if level < self.L and self.steps[level] % self.pb.regrid_interval == 0:
            self.regrid_from(level)
        child = self.levels.get(level + 1)
        has_child = child is not None and len(self.layout.get(level + 1, _EMPTY)) > 0
        fuse = self.fuse_sibling_fill and not has_child
        self.fill_level_ghosts(level, t0, siblings=not fuse)
        self.levels[level].fused_frame = fuse   # the finite check reads its sibling cells via the plan
        ev = None
        if has_child:
            # (ii) the full shadows (parents of the children), frames just
            # filled at t0.  A childless level skips (ii): its shadows are
            # ring-only and unchanged since (i).  With overlap_refresh the
            # exchange runs on its own stream while the step runs (the step
            # reads owned frames and sibling interiors only); the t1 fill
            # and the children's fills (stash = this buffer) wait for it.
            if self.overlap_refresh:
                self._xstream.wait_stream(self.stream)
                self._refresh(level, full_only=True, stream=self._xstream)  # (ii)
                ev = torch.cuda.Event()
                ev.record(self._xstream)
            else:
                self._refresh(level, full_only=True)                       # (ii)
        pool = self.levels[level]
        self._step_patches(level, dt, fused_siblings=fuse)
        self.steps[level] += 1
        t1 = t0 + dt
        pool.time = t1
        if has_child:
            if ev is not None:
                self.stream.wait_event(ev)
            # (iii) in two halves around the t1 fill.  The fill copies
            # sibling interiors into owned frames, and a boundary condition
            # corner outside the domain is built from such a copied cell;
            # the children's fills read that corner (through the ghost owner
            # map) when their parent stencil leaves the domain next to a
            # foreign sibling.  So the shadows' interiors must be at t1
            # before the fill, and the parents' frames go out after it.
            self._refresh(level)                                        # (iii-a)
            self.fill_level_ghosts(level, t1)
            self._refresh(level, full_only=True)                        # (iii-b)
            self._stash[level] = (t0, dt, pool.other)
            s = self.spec(level)
            dtf = dt / s.r_t
            for k in range(s.r_t):
                self.advance_level(level + 1, dtf, t0 + k * dtf)
            self.levels[level + 1].time = t1
            self._refresh(level + 1, coarsen=True)                      # (iv)
            self._average_down(level)
            del self._stash[level]

    def _advance_finest_overlapped(self, level: int, dt: float, t0: float) -> None:
        """The finest level with its shadow refresh (i) on the exchange stream:
        the parent-interpolated part of the fill and the tiles whose step
        reads no shadow run while the exchange is in flight; the BC patches'
        fill and the remaining tiles wait for it.  Same arithmetic as the
        sequential order (the two parts write disjoint cells)."""
        n1 = self._split_tiles(level)
        self._xstream.wait_stream(self.stream)
        self._refresh(level, stream=self._xstream)                     # (i)
        ev = torch.cuda.Event()
        ev.record(self._xstream)
        self.fill_level_ghosts(level, t0, siblings=False, part="interp")
        self.levels[level].fused_frame = True

        def between():
            self.stream.wait_event(ev)
            self.fill_level_ghosts(level, t0, siblings=False, part="bc")

        pool = self.levels[level]
        self._step_patches(level, dt, fused_siblings=True, split=(n1, between))
        self.steps[level] += 1
        pool.time = t0 + dt

    def owned_fields(self, level: int):
        """{global index: (box, h, hu, hv, bathy)} of this rank's patches."""
        pool = self.levels[level]
        host = pool.download()
        out = {}
        for p in range(pool.P):
            if pool.owned is not None and not pool.owned[p]:
                continue
            h, hu, hv, b = pool.patch_arrays(p, host=host)
            out[int(pool.gidx[p])] = (tuple(int(v) for v in pool.boxes[p]), h, hu, hv, b)
        return out
