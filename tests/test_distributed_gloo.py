"""Multi-rank host logic of the sharded path (distributed.py) with the gloo
backend on CPU, world sizes 2 and 4: SFC partition, shadow rules, transfer plans
and the whole-patch exchange (with host tensors standing in for device
pools; the CUDA pack kernel is exercised by tests/test_gpu_sharded.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _layouts():
    """A 3-level layout on a 64^2 level-1 grid, r=4: level-2/3 boxes chopped
    from a few blobs (deterministic)."""
    rng = np.random.default_rng(5)
    L2 = []
    for j in range(8, 56, 8):
        for i in range(4, 60, 8):
            if rng.random() < 0.6:
                L2.append((4 * i, 4 * j, 4 * i + 31, 4 * j + 31))
    L2 = np.array(sorted(L2, key=lambda b: (b[1], b[0])), np.int64)
    L3 = []
    for b in L2[::2]:
        for dj in (0, 64):
            for di in (0, 64):
                L3.append((4 * b[0] + 16 + di, 4 * b[1] + 16 + dj, 4 * b[0] + 16 + di + 47, 4 * b[1] + 16 + dj + 47))
    L3 = np.array(sorted(L3, key=lambda b: (b[1], b[0])), np.int64)
    return {1: np.array([[0, 0, 63, 63]], np.int64), 2: L2, 3: L3}


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1803_01450_b200.distributed import (Comm, needed, partition, patch_sizes, plan_acquire,
                                                       plan_refresh, ring_segments, run_transfer)
        comm = Comm()
        assert comm.world == world and comm.rank == rank
        comm.warmup_p2p(torch.device("cpu"))   # every rank in the first batch_isend_irecv
        layouts = _layouts()
        ratios = {1: (4, 4), 2: (4, 4), 3: (1, 1)}
        owners = {1: np.zeros(1, np.int32), 2: partition(layouts[2], 4, 4, world),
                  3: partition(layouts[3], 1, 1, world)}
        held = {lv: {r: needed(lv, r, layouts, owners, ratios) for r in range(world)} for lv in (1, 2, 3)}
        full = {lv: {r: needed(lv, r, layouts, owners, ratios, full_only=True) for r in range(world)}
                for lv in (1, 2, 3)}
        M3 = 6
        results = {}
        for lv in (2, 3):
            for use_ring in (False, True):
                B = layouts[lv]
                sizes = patch_sizes(B)
                rp, rro, rln, rsize = ring_segments(B)
                mine = held[lv][rank]
                offs = np.concatenate([[0], np.cumsum(sizes[mine])[:-1]]).astype(np.int64)
                FS = int(sizes[mine].sum()) + 1
                pool = torch.full((M3, FS), -1.0, dtype=torch.float64)
                for k, g in enumerate(mine):
                    if owners[lv][g] == rank:   # owners know their data: a function of (g, plane, cell)
                        vals = g * 1000.0 + torch.arange(M3 * int(sizes[g]), dtype=torch.float64).reshape(M3, -1)
                        pool[:, offs[k]:offs[k] + sizes[g]] = vals
                loc = {int(g): int(o) for g, o in zip(mine, offs)}

                def runs(gg, ring):
                    if not ring:
                        return [(0, int(sizes[gg]))]
                    sel = rp == gg
                    return list(zip(rro[sel].tolist(), rln[sel].tolist()))

                def nsz(g, ring):
                    r = np.zeros(len(g), bool) if ring is None else ring
                    return np.where(r, rsize[g], sizes[g])

                def pack(g, ring, src_off, buf):
                    n = int(nsz(g, ring).sum())
                    b2 = buf.view(M3, n)
                    at = 0
                    for i, (gg, so) in enumerate(zip(g, src_off)):
                        for (o, ln) in runs(gg, ring is not None and ring[i]):
                            b2[:, at:at + ln] = pool[:, so + o:so + o + ln]
                            at += ln

                def unpack(g, ring, buf, dst_off):
                    n = int(nsz(g, ring).sum())
                    b2 = buf.view(M3, n)
                    at = 0
                    for i, (gg, do) in enumerate(zip(g, dst_off)):
                        for (o, ln) in runs(gg, ring is not None and ring[i]):
                            pool[:, do + o:do + o + ln] = b2[:, at:at + ln]
                            at += ln

                offs_of = lambda g: np.array([loc[int(x)] for x in g], np.int64)
                tr = plan_refresh(rank, world, held[lv], owners[lv], full[lv] if use_ring else None)
                run_transfer(comm, tr, nsz, M3, offs_of, offs_of, pack, unpack, torch.float64, "cpu")
                ok, nring = True, 0
                for k, g in enumerate(mine):
                    vals = g * 1000.0 + torch.arange(M3 * int(sizes[g]), dtype=torch.float64).reshape(M3, -1)
                    got = pool[:, offs[k]:offs[k] + sizes[g]]
                    if use_ring and g not in full[lv][rank]:
                        nring += 1
                        for (o, ln) in runs(g, True):
                            ok &= bool(torch.equal(got[:, o:o + ln], vals[:, o:o + ln]))
                    else:
                        ok &= bool(torch.equal(got, vals))
                results[(lv, use_ring)] = (ok, len(mine), int((owners[lv][mine] == rank).sum()), nring)
        # acquire plan symmetry: what rank r receives from s equals what s sends to r
        want = {r: np.union1d(held[3][r], np.arange(min(3, len(layouts[3])))) for r in range(world)}
        tr = plan_acquire(rank, world, held[3], want, owners[3])
        sent = {q: g.tolist() for q, g in tr.send.items()}
        recv = {q: g.tolist() for q, g in tr.recv.items()}
        t = torch.tensor([comm.allreduce(torch.ones(1)).item()])
        # flag bits: a uint8 MAX all-reduce in place is the union of the
        # ranks' owned bits (sharded._reduce_flag_bits)
        bits = torch.zeros(64, dtype=torch.uint8)
        bits[rank::world] = 1 << (rank % 8)
        comm.allreduce(bits, dist.ReduceOp.MAX)
        want = torch.tensor([1 << (k % world % 8) for k in range(64)], dtype=torch.uint8)
        assert torch.equal(bits, want), bits
        q.put((rank, results, sent, recv, t.item()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_exchange(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, res, sent, recv, t = q.get(timeout=120)
        out[r] = (res, sent, recv, t)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shadows = {2: 0, 3: 0}
    rings = 0
    for r in range(world):
        res, sent, recv, t = out[r]
        assert t == world
        for (lv, use_ring), (ok, held_n, owned_n, nring) in res.items():
            assert ok, (r, lv, use_ring)
            assert owned_n > 0, (r, lv)
            if not use_ring:
                shadows[lv] += held_n - owned_n
            rings += nring
    assert all(v > 0 for v in shadows.values()), shadows   # the exchange had work to do
    assert rings > 0                                          # sibling-only shadows moved as rings
    # plans are mutually consistent
    for r in range(world):
        for s_ in range(world):
            if r == s_:
                continue
            assert out[r][1].get(s_, []) == out[s_][2].get(r, [])


def test_partition_balance_and_locality():
    from paper_1803_01450_b200.distributed import morton, partition
    assert morton(np.array([1]), np.array([0]))[0] == 1 and morton(np.array([0]), np.array([1]))[0] == 2
    g = np.arange(0, 1024, 32)
    I, J = np.meshgrid(g, g)
    B = np.stack([I.ravel(), J.ravel(), I.ravel() + 31, J.ravel() + 31], 1)
    for world in (2, 4, 8):
        own = partition(B, 1, 1, world)
        cnt = np.bincount(own, minlength=world)
        assert cnt.max() - cnt.min() <= 1
        # Z-order spans of a square grid are compact: each rank's bounding box is
        # at most twice its share of the area
        for r in range(world):
            b = B[own == r]
            area = (b[:, 2].max() - b[:, 0].min() + 1) * (b[:, 3].max() - b[:, 1].min() + 1)
            assert area <= 2.0 * 1024 * 1024 / world


def test_tiled_level1_shadow_sets():
    """Level 1 cut into tiles and spread over the ranks (sharded.py;
    Simulation.level1_boxes): the tiles cover the domain exactly once, every
    rank owns a share, and a rank holds -- besides its own tiles -- the
    sibling tiles within its frames and every tile under the parent
    stencils of its level-2 patches (so no rank needs all of level 1)."""
    from paper_1803_01450_b200.distributed import G, coarsen_floor, grow, needed, partition
    from paper_1803_01450_b200.regrid import chop_boxes
    lay = _layouts()
    full = lay[1]
    tiles = np.asarray(chop_boxes(full.astype(np.int32), 16, 16, aligned=True), np.int64).reshape(-1, 4)
    cover = np.zeros((64, 64), int)
    for b in tiles:
        assert b[0] % 16 == 0 and b[1] % 16 == 0
        cover[b[1]:b[3] + 1, b[0]:b[2] + 1] += 1
    assert len(tiles) == 16 and (cover == 1).all()
    lay = dict(lay)
    lay[1] = tiles
    R = {1: (4, 4), 2: (4, 4)}
    for world in (2, 4):
        own = {lev: partition(b, 4 ** (3 - lev), 4 ** (3 - lev), world) for lev, b in lay.items()}
        assert set(own[1]) == set(range(world))
        fewer = False
        for r in range(world):
            held = needed(1, r, lay, own, R)
            mine = np.flatnonzero(own[1] == r)
            assert set(mine) <= set(held)
            # every level-1 tile meeting the stencil of an owned level-2 patch
            F = lay[2][own[2] == r]
            st = grow(coarsen_floor(grow(F, G), 4, 4), 1)
            for k, t in enumerate(tiles):
                g = grow(t[None], G)[0]
                hit = ((st[:, 0] <= g[2]) & (st[:, 2] >= g[0]) & (st[:, 1] <= g[3]) & (st[:, 3] >= g[1])).any()
                if hit:
                    assert k in held, (world, r, k)
            fewer |= len(held) < len(tiles)
        assert fewer or world == 2
