"""Simulation frames written straight from the device pools, plus the
reader and the frame differ.

The file format is the reference's (frames.py:1-27 of
/root/reference/pkg/src/mlamr): an ASCII header with C99 hexfloat numbers,
then one record per patch, levels ascending and patches in list order.  A
binary record is five little-endian int64 (level, lo_i, lo_j, hi_i, hi_j)
followed by the interior planes bathymetry, h_0, hu_0, hv_0, h_1, ... as
row-major float64 (x fastest); the text form writes a ``patch`` line and
``ny`` comma-separated hexfloat rows per plane.

``mlamr_pack_frame`` builds each level's binary records in HBM (header
words included), so a binary frame is one device-to-host copy into pinned
memory and one file write.  Under sharding every rank packs the records of
the patches it owns and rank 0 assembles the file in global patch order.
``tests/test_gpu_frames.py`` checks the bytes against frames the reference
itself wrote for the same run (tests/golden/frames_shelf_small.npz).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch

FORMAT_VERSION = 1
MAGIC_BINARY = "MLAMR FRAME"
MAGIC_TEXT = "MLAMR FRAME-TEXT"
_REC_HDR = struct.Struct("<5q")


from .errors import FrameFormatError  # noqa: E402,F401  (the reference's class when importable)


# -- writing ------------------------------------------------------------------------------
def header_text(time: float, num_layers: int, domain, rest, levels, num_patches: int,
                text_mode: bool) -> str:
    """Header lines (frames.py:103-118): ``levels`` = [(level, nx, ny, dx, dy)]."""
    lines = [
        f"{MAGIC_TEXT if text_mode else MAGIC_BINARY} {FORMAT_VERSION}",
        f"time {float(time).hex()}",
        f"num_layers {num_layers}",
        f"num_levels {len(levels)}",
        "domain " + " ".join(float(v).hex() for v in domain),
        "rest " + " ".join(float(v).hex() for v in rest),
    ]
    lines += [f"level {lv} {nx} {ny} {float(dx).hex()} {float(dy).hex()}" for lv, nx, ny, dx, dy in levels]
    lines += [f"num_patches {num_patches}", "end_header"]
    return "\n".join(lines) + "\n"


def _record_layout(boxes: np.ndarray, M: int):
    """Element offsets (8-byte units) of each patch record and the total."""
    if len(boxes) == 0:
        return np.zeros(0, np.int64), 0
    n = (boxes[:, 2] - boxes[:, 0] + 1).astype(np.int64) * (boxes[:, 3] - boxes[:, 1] + 1)
    size = 5 + (1 + 3 * M) * n
    off = np.zeros(len(boxes), np.int64)
    off[1:] = np.cumsum(size)[:-1]
    return off, int(size.sum())


def _pack(sim, level: int, pool, rec_off_local: np.ndarray, total: int, plist=None) -> torch.Tensor:
    """Device body of one level's records; ``plist`` = local patch indices."""
    from .device import arena
    upload = arena().upload
    with torch.cuda.stream(sim.stream):
        out = torch.empty(max(total, 1), dtype=torch.float64, device=sim.dev)
    if total == 0:
        return out[:0]
    off_d = upload(rec_off_local, sim.dev, sim.stream)
    pl_d = upload(np.asarray(plist, np.int32), sim.dev, sim.stream) if plist is not None else None
    n_list = len(plist) if plist is not None else pool.P
    bpp = max(1, min(64, (pool.max_interior + 255) // 256))
    sim._call(sim.lib.mlamr_pack_frame, pool.struct(), pool.state.data_ptr(), level, off_d.data_ptr(),
              pl_d.data_ptr() if pl_d is not None else None, n_list, bpp, out.data_ptr(), sim.sh)
    sim._keep_frame = (off_d, pl_d)
    return out[:total]


def _level_meta(sim):
    return [(s.level, s.nx, s.ny, s.dx, s.dy) for s in sim.specs]


def _global_boxes(sim, level: int) -> np.ndarray:
    layout = getattr(sim, "layout", None)
    if layout is not None:
        return np.asarray(layout.get(level, np.zeros((0, 4), np.int64)))
    pool = sim.levels.get(level)
    return pool.boxes if pool is not None else np.zeros((0, 4), np.int64)


def frame_body(sim) -> tuple[int, np.ndarray | None]:
    """(num_patches, binary body as uint8) of the current hierarchy.  On a
    sharded run rank 0 gets the assembled body, other ranks None."""
    M = sim.M
    comm = getattr(sim, "comm", None)
    sharded = comm is not None and comm.world > 1
    parts, n_total = [], 0
    for s in sim.specs:
        lev = s.level
        boxes = _global_boxes(sim, lev)
        n_total += len(boxes)
        if len(boxes) == 0:
            continue
        pool = sim.levels[lev]
        g_off, g_total = _record_layout(boxes, M)
        if not sharded:
            body = _pack(sim, lev, pool, g_off, g_total)
            host = torch.empty(g_total, dtype=torch.float64, pin_memory=True)
            with torch.cuda.stream(sim.stream):
                host.copy_(body, non_blocking=True)
            parts.append(host)
            continue
        parts.append(_gather_level(sim, lev, pool, boxes, M))
    sim.stream.synchronize()
    if sharded and comm.rank != 0:
        return n_total, None
    blob = [p.numpy().view(np.uint8) for p in parts]
    sim.d2h_bytes += sum(b.size for b in blob)
    return n_total, (np.concatenate(blob) if blob else np.zeros(0, np.uint8))


def _gather_level(sim, lev, pool, boxes, M):
    """Sharded: each rank packs its owned records (global order, compact);
    rank 0 receives every rank's block and scatters records into place."""
    comm = sim.comm
    owner = np.asarray(sim.owner[lev])
    n = (boxes[:, 2] - boxes[:, 0] + 1).astype(np.int64) * (boxes[:, 3] - boxes[:, 1] + 1)
    size = 5 + (1 + 3 * M) * n
    mine_g = np.flatnonzero(owner == comm.rank)
    local = np.array([pool.local_of(int(g)) for g in mine_g], np.int32)
    c_off = np.zeros(pool.P, np.int64)
    c_off[local] = np.concatenate([[0], np.cumsum(size[mine_g])[:-1]]) if len(mine_g) else []
    body = _pack(sim, lev, pool, c_off, int(size[mine_g].sum()), plist=local if len(local) else None)
    sim.stream.synchronize()
    g_off, g_total = _record_layout(boxes, M)
    if comm.rank != 0:
        comm.exchange({0: body.contiguous()} if body.numel() else {}, {})
        return torch.zeros(0, dtype=torch.float64)
    recvs = {}
    for q in range(1, comm.world):
        cnt = int(size[owner == q].sum())
        recvs[q] = torch.empty(cnt, dtype=torch.float64, device=sim.dev)
    comm.exchange({}, {q: t for q, t in recvs.items() if t.numel()})
    out = np.empty(g_total, np.float64)
    blocks = {0: body.cpu().numpy()}
    blocks.update({q: t.cpu().numpy() for q, t in recvs.items()})
    for q, blk in blocks.items():
        pos = 0
        for g in np.flatnonzero(owner == q):
            out[g_off[g]:g_off[g] + size[g]] = blk[pos:pos + size[g]]
            pos += size[g]
    return torch.from_numpy(out)


def _text_records(body: np.ndarray, boxes_all, M: int) -> str:
    parts = []
    words = body.view(np.float64)
    ints = body.view(np.int64)
    pos = 0
    for _ in range(len(boxes_all)):
        lev, lo_i, lo_j, hi_i, hi_j = (int(v) for v in ints[pos:pos + 5])
        pos += 5
        nx, ny = hi_i - lo_i + 1, hi_j - lo_j + 1
        parts.append(f"patch {lev} {lo_i} {lo_j} {hi_i} {hi_j}\n")
        for _f in range(1 + 3 * M):
            plane = words[pos:pos + nx * ny].reshape(ny, nx)
            pos += nx * ny
            parts.extend(",".join(float(v).hex() for v in row) + "\n" for row in plane)
    return "".join(parts)


def frame_bytes(sim, text_mode: bool = False, time: float | None = None) -> bytes | None:
    """The frame file's bytes (None on non-zero ranks of a sharded run)."""
    pb = sim.pb
    n_patches, body = frame_body(sim)
    if body is None:
        return None
    head = header_text(sim.time if time is None else time, sim.M, pb.domain, pb.eta_rest, _level_meta(sim),
                       n_patches, text_mode).encode("ascii")
    if not text_mode:
        return head + body.tobytes()
    boxes_all = [b for s in sim.specs for b in _global_boxes(sim, s.level)]
    return head + _text_records(body, boxes_all, sim.M).encode("ascii")


def write_frame(sim, path, text_mode: bool = False, time: float | None = None) -> None:
    """Write the current hierarchy as a reference frame file (rank 0 writes)."""
    data = frame_bytes(sim, text_mode, time)
    if data is not None:
        with open(path, "wb") as f:
            f.write(data)


# -- reading and comparing (frames.py:166-323 of the reference) ----------------------------
@dataclass
class FramePatch:
    level: int
    box: tuple
    bathy: np.ndarray
    h: np.ndarray
    hu: np.ndarray
    hv: np.ndarray


@dataclass
class Frame:
    version: int
    time: float
    num_layers: int
    domain: tuple
    rest: tuple
    levels: list
    patches: list

    def level_meta(self, level: int):
        for meta in self.levels:
            if meta[0] == level:
                return meta
        raise FrameFormatError(f"frame has no level {level}")


def _parse_header(text: str, path):
    lines = text.splitlines()
    first = lines[0].split() if lines else []
    if len(first) != 3 or first[0] != "MLAMR":
        raise FrameFormatError(f"{path}: not a frame file")
    magic = f"{first[0]} {first[1]}"
    if magic not in (MAGIC_BINARY, MAGIC_TEXT):
        raise FrameFormatError(f"{path}: unknown magic {magic!r}")
    if int(first[2]) != FORMAT_VERSION:
        raise FrameFormatError(f"{path}: format version {first[2]} not supported")
    meta = {"levels": []}
    parsers = {
        "time": lambda t: float.fromhex(t[0]),
        "num_layers": lambda t: int(t[0]),
        "num_levels": lambda t: int(t[0]),
        "domain": lambda t: tuple(float.fromhex(v) for v in t[:4]),
        "rest": lambda t: tuple(float.fromhex(v) for v in t),
        "num_patches": lambda t: int(t[0]),
    }
    for line in lines[1:]:
        tok = line.split()
        if not tok:
            continue
        if tok[0] == "level":
            meta["levels"].append((int(tok[1]), int(tok[2]), int(tok[3]), float.fromhex(tok[4]),
                                   float.fromhex(tok[5])))
        elif tok[0] in parsers:
            meta[tok[0]] = parsers[tok[0]](tok[1:])
        else:
            raise FrameFormatError(f"{path}: unknown header line {line!r}")
    need = ("time", "num_layers", "num_levels", "domain", "rest", "num_patches")
    if any(k not in meta for k in need) or len(meta["levels"]) != meta["num_levels"]:
        raise FrameFormatError(f"{path}: incomplete header")
    return meta, magic == MAGIC_TEXT


def parse_frame(blob: bytes, path="<bytes>") -> Frame:
    marker = b"end_header\n"
    pos = blob.find(marker)
    if pos < 0:
        raise FrameFormatError(f"{path}: missing end_header")
    meta, text = _parse_header(blob[:pos].decode("ascii", errors="replace"), path)
    body = blob[pos + len(marker):]
    M = meta["num_layers"]
    nf = 1 + 3 * M
    patches = []
    if text:
        rows = body.decode("ascii").splitlines()
        k = 0
        for _ in range(meta["num_patches"]):
            tok = rows[k].split()
            if tok[0] != "patch":
                raise FrameFormatError(f"{path}: expected a patch line")
            k += 1
            lev, lo_i, lo_j, hi_i, hi_j = (int(v) for v in tok[1:6])
            ny = hi_j - lo_j + 1
            fields = []
            for _f in range(nf):
                fields.append(np.array([[float.fromhex(v) for v in rows[k + j].split(",")] for j in range(ny)]))
                k += ny
            patches.append(_assemble(lev, (lo_i, lo_j, hi_i, hi_j), fields, M))
    else:
        off = 0
        for _ in range(meta["num_patches"]):
            lev, lo_i, lo_j, hi_i, hi_j = _REC_HDR.unpack_from(body, off)
            off += _REC_HDR.size
            nx, ny = hi_i - lo_i + 1, hi_j - lo_j + 1
            fields = []
            for _f in range(nf):
                fields.append(np.frombuffer(body, "<f8", nx * ny, off).reshape(ny, nx).copy())
                off += 8 * nx * ny
            patches.append(_assemble(lev, (lo_i, lo_j, hi_i, hi_j), fields, M))
    return Frame(FORMAT_VERSION, meta["time"], M, meta["domain"], meta["rest"], meta["levels"], patches)


def read_frame(path) -> Frame:
    with open(path, "rb") as f:
        return parse_frame(f.read(), path)


def _assemble(lev, box, fields, M) -> FramePatch:
    return FramePatch(lev, box, fields[0], np.stack(fields[1::3][:M]), np.stack(fields[2::3][:M]),
                      np.stack(fields[3::3][:M]))


def composite_fields(frame: Frame) -> dict:
    """The hierarchy flattened onto the finest grid, finer data winning."""
    _, nxf, nyf, _, _ = frame.levels[-1]
    M = frame.num_layers
    out = {"bathy": np.full((nyf, nxf), np.nan)}
    for k in ("h", "hu", "hv"):
        out[k] = np.full((M, nyf, nxf), np.nan)
    for p in sorted(frame.patches, key=lambda q: q.level):
        _, nxl, nyl, _, _ = frame.level_meta(p.level)
        fx, rx = divmod(nxf, nxl)
        fy, ry = divmod(nyf, nyl)
        if rx or ry:
            raise FrameFormatError(f"level {p.level} grid does not divide the finest grid")
        lo_i, lo_j, hi_i, hi_j = p.box
        sl = (slice(lo_j * fy, (hi_j + 1) * fy), slice(lo_i * fx, (hi_i + 1) * fx))
        up = lambda a: np.repeat(np.repeat(a, fy, axis=-2), fx, axis=-1)  # noqa: E731
        out["bathy"][sl] = up(p.bathy)
        for k in ("h", "hu", "hv"):
            out[k][(slice(None),) + sl] = up(getattr(p, k))
    if np.isnan(out["bathy"]).any():
        raise FrameFormatError("frame does not cover the domain")
    out["eta"] = np.cumsum(out["h"][::-1], axis=0)[::-1] + out["bathy"]
    return out


def l1_diff(a: Frame, b: Frame) -> dict:
    """Mean and max |difference| of layer surfaces and depths on the finer
    of the two finest grids (the reference's ``compare``)."""
    if a.domain != b.domain or a.num_layers != b.num_layers:
        raise FrameFormatError("frames differ in domain or layer count")
    fa, fb = composite_fields(a), composite_fields(b)
    if fa["h"].shape != fb["h"].shape:
        if fa["h"].shape[1] < fb["h"].shape[1]:
            fa, fb = fb, fa
        fy, ry = divmod(fa["h"].shape[1], fb["h"].shape[1])
        fx, rx = divmod(fa["h"].shape[2], fb["h"].shape[2])
        if rx or ry:
            raise FrameFormatError("frame resolutions are not nested")
        for k in ("h", "eta"):
            fb[k] = np.repeat(np.repeat(fb[k], fy, axis=-2), fx, axis=-1)
    out = {}
    for k in ("eta", "h"):
        d = np.abs(fa[k] - fb[k])
        for m in range(d.shape[0]):
            out[f"{k}_{m + 1}_l1"] = float(d[m].mean())
            out[f"{k}_{m + 1}_linf"] = float(d[m].max())
    return out


def main(argv=None) -> int:
    import argparse
    import json
    ap = argparse.ArgumentParser(description="compare two MLAMR frame files")
    ap.add_argument("a")
    ap.add_argument("b")
    args = ap.parse_args(argv)
    print(json.dumps(l1_diff(read_frame(args.a), read_frame(args.b)), indent=1, sort_keys=True))
    return 0


if __name__ == "__main__":  # pragma: no cover
    raise SystemExit(main())
