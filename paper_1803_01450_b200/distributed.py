"""Patch sharding across GPUs.

Every rank holds the full patch tables (boxes) of every level.  Layouts
are computed redundantly and deterministically from all-reduced flags.
Each rank stores state only for the patches it **owns** plus **shadow**
replicas of foreign patches its kernels read:

1. *siblings*: patches whose interior meets the 2-cell frame of an owned
   patch of the same level (ghost.py:186-196);
2. *parents*: patches of level l whose interior or frame meets the
   interpolation stencil of an owned level-(l+1) patch's ghost bands or
   refined cells: coarsen(box grown by 2) grown by 1 (ghost.py:170-185,
   gather pass 2 included);
3. *children*: patches of level l+1 whose coarse footprint meets an owned
   level-l patch (coarsen.py:57-75): the coarse owner does the averaging.

Shadows are refreshed by whole-patch copies from their owners at fixed
points of the level recursion (driver.Simulation); a shadow is never
written by its holder.  Ownership is a Morton (Z-order) space-filling
curve over patch lower corners in the finest level's index space, cut into
equal-cell spans per level, so parents and children mostly share a rank.

The exchange is one grouped send/recv per level (NCCL over NVLink on GPU;
gloo tests stage through host memory).  dt, flags, composite mass and the
finite check are all-reduces.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Dict, List, Optional

import numpy as np
import torch
import torch.distributed as dist

G = 2  # ghost width


# ---------------------------------------------------------------------------
# space-filling curve partition
# ---------------------------------------------------------------------------
def _spread(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.uint64) & np.uint64(0xFFFFFFFF)
    v = (v | (v << np.uint64(16))) & np.uint64(0x0000FFFF0000FFFF)
    v = (v | (v << np.uint64(8))) & np.uint64(0x00FF00FF00FF00FF)
    v = (v | (v << np.uint64(4))) & np.uint64(0x0F0F0F0F0F0F0F0F)
    v = (v | (v << np.uint64(2))) & np.uint64(0x3333333333333333)
    v = (v | (v << np.uint64(1))) & np.uint64(0x5555555555555555)
    return v


def morton(i: np.ndarray, j: np.ndarray) -> np.ndarray:
    """Z-order key of non-negative integer coordinates."""
    return _spread(np.asarray(i)) | (_spread(np.asarray(j)) << np.uint64(1))


def partition(boxes: np.ndarray, scale_x: int, scale_y: int, world: int) -> np.ndarray:
    """Owner rank per patch: Morton order of the lower corners (scaled to
    the finest level), cut into `world` spans of equal cell count."""
    P = len(boxes)
    if P == 0 or world == 1:
        return np.zeros(P, dtype=np.int32)
    b = np.asarray(boxes, dtype=np.int64)
    key = morton(np.maximum(b[:, 0], 0) * scale_x, np.maximum(b[:, 1], 0) * scale_y)
    order = np.lexsort((np.arange(P), key))
    cells = ((b[:, 2] - b[:, 0] + 1) * (b[:, 3] - b[:, 1] + 1)).astype(np.float64)
    c = cells[order]
    mid = np.cumsum(c) - 0.5 * c
    owner = np.empty(P, dtype=np.int32)
    owner[order] = np.minimum(world - 1, (mid * world / c.sum()).astype(np.int64))
    return owner


# ---------------------------------------------------------------------------
# shadow rules
# ---------------------------------------------------------------------------
def _meets(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Pairwise box intersection test, a [n,4] x b [m,4] -> bool [n,m]."""
    if len(a) == 0 or len(b) == 0:
        return np.zeros((len(a), len(b)), bool)
    return ((a[:, None, 0] <= b[None, :, 2]) & (b[None, :, 0] <= a[:, None, 2]) &
            (a[:, None, 1] <= b[None, :, 3]) & (b[None, :, 1] <= a[:, None, 3]))


def _any_meet(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """For each box of a: does it meet any box of b?  (native bucket grid)."""
    from . import _native as N
    a = np.ascontiguousarray(a, dtype=np.int64).reshape(-1, 4)
    b = np.ascontiguousarray(b, dtype=np.int64).reshape(-1, 4)
    out = np.zeros(len(a), dtype=np.uint8)
    if len(a) == 0 or len(b) == 0:
        return out.astype(bool)
    span = max(int((b[:, 2] - b[:, 0]).max()), int((b[:, 3] - b[:, 1]).max())) + 1
    rc = N.lib().mlamr_boxes_meet_any(a.ctypes.data, len(a), b.ctypes.data, len(b), max(16, span), out.ctypes.data)
    if rc != 0:
        return _meets(a, b).any(axis=1)
    return out.astype(bool)


def grow(b: np.ndarray, w: int) -> np.ndarray:
    return b + np.array([-w, -w, w, w], dtype=np.int64)


def coarsen_floor(b: np.ndarray, rx: int, ry: int) -> np.ndarray:
    """Coarse cells containing any cell of b (floor division, any alignment)."""
    return np.stack([np.floor_divide(b[:, 0], rx), np.floor_divide(b[:, 1], ry),
                     np.floor_divide(b[:, 2], rx), np.floor_divide(b[:, 3], ry)], axis=1)


def needed(level: int, rank: int, layouts: Dict[int, np.ndarray], owners: Dict[int, np.ndarray],
           ratios: Dict[int, tuple], extra_fine: Optional[Dict[int, np.ndarray]] = None,
           full_only: bool = False, with_children: bool = True) -> np.ndarray:
    """Sorted global indices of level `level` patches rank `rank` must hold
    (owned + shadows).  ratios[l] = (r_x, r_y) between l and l+1.
    ``extra_fine[l+1]`` adds fine boxes (e.g. old layouts during a regrid)
    whose parent stencils must be present on this level.

    ``full_only``: only the patches that must be held in full -- owned,
    parents and (``with_children``) children.  The rest are sibling-only
    shadows: the ghost fill of owned patches reads nothing of them but the
    interior ring within two cells of their boundary, which is all a
    refresh sends.  Children are read in full only by the coarsening, so
    only the refresh in front of it sends them whole."""
    B = layouts.get(level)
    if B is None or len(B) == 0:
        return np.zeros(0, np.int64)
    B = np.asarray(B, np.int64)
    own = owners[level] == rank
    need = own.copy()
    mine = B[own]
    # 1. siblings: interiors meeting an owned patch's frame
    if not full_only:
        need |= _any_meet(B, grow(mine, G))
    # 2. parents of owned (and extra) finer patches: full boxes meeting the stencil
    fine = []
    if level + 1 in layouts and len(layouts[level + 1]):
        F = np.asarray(layouts[level + 1], np.int64)
        fine.append(F[owners[level + 1] == rank])
    if extra_fine and level + 1 in extra_fine:
        fine.append(np.asarray(extra_fine[level + 1], np.int64))
    if fine:
        F = np.concatenate(fine)
        if len(F):
            rx, ry = ratios[level]
            stencil = grow(coarsen_floor(grow(F, G), rx, ry), 1)
            need |= _any_meet(grow(B, G), stencil)
    # 3. children: finer patches averaged onto owned coarse patches -- the
    # coarse owner needs them; on this level, the patches whose coarse
    # footprint meets an owned patch of level-1
    if (with_children or not full_only) and level - 1 in layouts and len(layouts[level - 1]):
        C = np.asarray(layouts[level - 1], np.int64)
        cown = C[owners[level - 1] == rank]
        rx, ry = ratios[level - 1]
        need |= _any_meet(coarsen_floor(B, rx, ry), cown)
    return np.flatnonzero(need).astype(np.int64)


# ---------------------------------------------------------------------------
# communication
# ---------------------------------------------------------------------------
class Comm:
    """torch.distributed wrapper; single-rank when not initialised."""

    def __init__(self):
        self.on = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank() if self.on else 0
        self.world = dist.get_world_size() if self.on else 1
        self.backend = dist.get_backend() if self.on else "none"

    @property
    def staged(self) -> bool:
        """gloo moves host tensors only: stage device tensors through host."""
        return self.backend == "gloo"

    def allreduce(self, t: torch.Tensor, op=None) -> torch.Tensor:
        if self.world == 1:
            return t
        op = op or dist.ReduceOp.SUM
        if self.staged and t.is_cuda:
            h = t.cpu()
            dist.all_reduce(h, op=op)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=op)
        return t

    def warmup_p2p(self, device) -> None:
        """One ring exchange in which every rank takes part.  With NCCL the
        first batch_isend_irecv of a group must involve all its ranks, and
        later exchanges skip ranks with nothing to move."""
        if self.world == 1:
            return
        dev = torch.device("cpu") if self.staged else device
        s = torch.full((1,), float(self.rank), dtype=torch.float64, device=dev)
        r = torch.empty(1, dtype=torch.float64, device=dev)
        ops = [dist.P2POp(dist.isend, s, (self.rank + 1) % self.world),
               dist.P2POp(dist.irecv, r, (self.rank - 1) % self.world)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()

    def exchange(self, sends: Dict[int, torch.Tensor], recvs: Dict[int, torch.Tensor]) -> None:
        """Grouped point-to-point transfer: sends[peer] -> peer, recvs[peer] <- peer."""
        if self.world == 1 or (not sends and not recvs):
            return
        if self.staged:
            s_host = {q: t.cpu() if t.is_cuda else t for q, t in sends.items()}
            r_host = {q: torch.empty(t.shape, dtype=t.dtype) if t.is_cuda else t for q, t in recvs.items()}
            ops = [dist.P2POp(dist.isend, s_host[q], q) for q in sorted(s_host)]
            ops += [dist.P2POp(dist.irecv, r_host[q], q) for q in sorted(r_host)]
            for w in dist.batch_isend_irecv(ops):
                w.wait()
            for q, t in recvs.items():
                if t.is_cuda:
                    t.copy_(r_host[q])
        else:
            ops = [dist.P2POp(dist.isend, sends[q], q) for q in sorted(sends)]
            ops += [dist.P2POp(dist.irecv, recvs[q], q) for q in sorted(recvs)]
            for w in dist.batch_isend_irecv(ops):
                w.wait()


@dataclass
class Transfer:
    """Which patches move between which ranks for one level: for each peer,
    the (sorted) global indices this rank sends and receives, and (refresh
    only) which of them move as the two-cell interior ring only."""
    send: Dict[int, np.ndarray]
    recv: Dict[int, np.ndarray]
    send_ring: Optional[Dict[int, np.ndarray]] = None
    recv_ring: Optional[Dict[int, np.ndarray]] = None


def plan_refresh(rank: int, world: int, held: Dict[int, np.ndarray], owner: np.ndarray,
                 full: Optional[Dict[int, np.ndarray]] = None) -> Transfer:
    """Shadow refresh: every rank receives each held foreign patch from its
    owner; `held[r]` = sorted global indices rank r holds (for all r).
    With `full[r]` (the patches rank r needs in full), the others move as
    their interior ring only."""
    send, recv, sring, rring = {}, {}, {}, {}
    mine = held[rank]
    for q in range(world):
        if q == rank:
            continue
        r = mine[owner[mine] == q]
        if len(r):
            recv[q] = r
            if full is not None:
                rring[q] = ~np.isin(r, full[rank])
        theirs = held[q]
        s = theirs[owner[theirs] == rank]
        if len(s):
            send[q] = s
            if full is not None:
                sring[q] = ~np.isin(s, full[q])
    if full is None:
        return Transfer(send, recv)
    return Transfer(send, recv, sring, rring)


def ring_segments(boxes: np.ndarray):
    """Per patch block ((ny+4) x (nx+4), ghost width 2): the two-cell
    interior ring as (relative offset, length) runs -- the two interior rows
    next to the bottom and top frame at full block width, then the two
    interior columns next to the left and right frame on the rows between.
    Patches too small for a distinct ring are whole blocks.  Returns
    (patch_index, rel_offset, length, packed_size_per_patch)."""
    b = np.asarray(boxes, np.int64).reshape(-1, 4)
    NX = b[:, 2] - b[:, 0] + 1 + 2 * G
    NY = b[:, 3] - b[:, 1] + 1 + 2 * G
    pi, ro, ln = [], [], []
    size = np.zeros(len(b), np.int64)
    small = (NX - 2 * G <= 4) | (NY - 2 * G <= 4)
    for k in np.flatnonzero(small):
        pi.append(np.array([k]))
        ro.append(np.array([0]))
        ln.append(np.array([NX[k] * NY[k]]))
        size[k] = NX[k] * NY[k]
    big = np.flatnonzero(~small)
    if len(big):
        nx_, ny_ = NX[big], NY[big]
        # the two full-width row runs
        pi += [big, big]
        ro += [2 * nx_, (ny_ - 4) * nx_]
        ln += [2 * nx_, 2 * nx_]
        # the side pairs on rows 4 .. NY-5
        nrow = ny_ - 8
        rep = np.repeat(np.arange(len(big)), nrow)
        start = np.concatenate([[0], np.cumsum(nrow)[:-1]])
        J = 4 + np.arange(int(nrow.sum())) - np.repeat(start, nrow)
        NXr = nx_[rep]
        pi += [big[rep], big[rep]]
        ro += [J * NXr + 2, J * NXr + NXr - 4]
        ln += [np.full(len(J), 2, np.int64), np.full(len(J), 2, np.int64)]
        size[big] = 4 * nx_ + 4 * nrow
    pi = np.concatenate(pi) if pi else np.zeros(0, np.int64)
    ro = np.concatenate(ro) if ro else np.zeros(0, np.int64)
    ln = np.concatenate(ln) if ln else np.zeros(0, np.int64)
    order = np.lexsort((ro, pi))
    return pi[order], ro[order], ln[order], size


def plan_acquire(rank: int, world: int, have: Dict[int, np.ndarray], want: Dict[int, np.ndarray],
                 owner: np.ndarray) -> Transfer:
    """Reshape: rank r receives want[r] \\ have[r] from the owners (which
    hold their owned patches)."""
    send, recv = {}, {}
    for q in range(world):
        miss_q = np.setdiff1d(want[q], have[q], assume_unique=True)
        if q == rank:
            for s in range(world):
                if s == rank:
                    continue
                r = miss_q[owner[miss_q] == s]
                if len(r):
                    recv[s] = r
        else:
            s_ = miss_q[owner[miss_q] == rank]
            if len(s_):
                send[q] = s_
    return Transfer(send, recv)


def patch_sizes(boxes: np.ndarray) -> np.ndarray:
    b = np.asarray(boxes, np.int64).reshape(-1, 4)
    return (b[:, 2] - b[:, 0] + 1 + 2 * G) * (b[:, 3] - b[:, 1] + 1 + 2 * G)


def run_transfer(comm: Comm, tr: Transfer, sizes: Callable, nplanes: int,
                 src_offsets: Callable[[np.ndarray], np.ndarray],
                 dst_offsets: Callable[[np.ndarray], np.ndarray],
                 pack: Callable, unpack: Callable, dtype, device) -> int:
    """Execute a Transfer: pack owned patch blocks (all planes) per peer,
    grouped send/recv, unpack into the holder's pool.  `sizes(gidx, ring)`
    gives the packed elements per patch; `pack(gidx, ring, src_off, buf)` /
    `unpack(gidx, ring, buf, dst_off)` move whole blocks, or their interior
    rings where `ring` is set, between a pool and a [nplanes, n] packed
    buffer.  Returns the bytes sent."""
    sends, recvs = {}, {}
    sent = 0
    for q, g in tr.send.items():
        ring = tr.send_ring[q] if tr.send_ring is not None else None
        n = int(sizes(g, ring).sum())
        buf = torch.empty(nplanes * n, dtype=dtype, device=device)
        pack(g, ring, src_offsets(g), buf)
        sends[q] = buf
        sent += buf.numel() * buf.element_size()
    for q, g in tr.recv.items():
        ring = tr.recv_ring[q] if tr.recv_ring is not None else None
        n = int(sizes(g, ring).sum())
        recvs[q] = torch.empty(nplanes * n, dtype=dtype, device=device)
    comm.exchange(sends, recvs)
    for q, g in tr.recv.items():
        ring = tr.recv_ring[q] if tr.recv_ring is not None else None
        unpack(g, ring, recvs[q], dst_offsets(g))
    return sent
