"""Index-space geometry (mesh.py:23-141 under /root/reference/pkg/src/mlamr).

Inclusive boxes in a level's global index space, the level ladder, and the
boolean morphology used by flagging and nesting.  Patch storage itself
lives on the device (:mod:`.device`); this module is host bookkeeping only.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple, Optional

import numpy as np

GHOST_WIDTH = 2


@dataclass(frozen=True)
class LevelSpec:
    """One level of the ladder and its ratios to the next finer level."""

    level: int
    nx: int
    ny: int
    dx: float
    dy: float
    r_x: int = 1
    r_y: int = 1
    r_t: int = 1


class IndexBox(NamedTuple):
    """Inclusive rectangle of cell indices (lo_i, lo_j, hi_i, hi_j)."""

    lo_i: int
    lo_j: int
    hi_i: int
    hi_j: int

    @property
    def nx(self) -> int:
        return self.hi_i - self.lo_i + 1

    @property
    def ny(self) -> int:
        return self.hi_j - self.lo_j + 1

    @property
    def ncells(self) -> int:
        return self.nx * self.ny

    def intersection(self, o: "IndexBox") -> Optional["IndexBox"]:
        a, b = max(self.lo_i, o.lo_i), max(self.lo_j, o.lo_j)
        c, d = min(self.hi_i, o.hi_i), min(self.hi_j, o.hi_j)
        return None if (c < a or d < b) else IndexBox(a, b, c, d)

    def contains_box(self, o: "IndexBox") -> bool:
        return (self.lo_i <= o.lo_i and self.lo_j <= o.lo_j
                and o.hi_i <= self.hi_i and o.hi_j <= self.hi_j)

    def grown(self, w: int) -> "IndexBox":
        return IndexBox(self.lo_i - w, self.lo_j - w, self.hi_i + w, self.hi_j + w)

    def refined(self, rx: int, ry: int) -> "IndexBox":
        return IndexBox(self.lo_i * rx, self.lo_j * ry, (self.hi_i + 1) * rx - 1, (self.hi_j + 1) * ry - 1)

    def coarsened(self, rx: int, ry: int) -> "IndexBox":
        if self.lo_i % rx or self.lo_j % ry or (self.hi_i + 1) % rx or (self.hi_j + 1) % ry:
            raise ValueError(f"{self} is not aligned to ratio ({rx},{ry})")
        return IndexBox(self.lo_i // rx, self.lo_j // ry, (self.hi_i + 1) // rx - 1, (self.hi_j + 1) // ry - 1)


def boxes_array(boxes) -> np.ndarray:
    return np.asarray([tuple(b) for b in boxes], dtype=np.int64).reshape(-1, 4)


def dilate(mask: np.ndarray, width: int) -> np.ndarray:
    """8-neighbour growth by ``width`` cells (mesh.py:116-127), as a
    separable max filter (identical result for a square structuring
    element)."""
    out = mask.astype(bool, copy=True)
    for _ in range(width):
        h = out.copy()
        h[:, 1:] |= out[:, :-1]
        h[:, :-1] |= out[:, 1:]
        v = h.copy()
        v[1:, :] |= h[:-1, :]
        v[:-1, :] |= h[1:, :]
        out = v
    return out


def erode(mask: np.ndarray, width: int) -> np.ndarray:
    """Shrink by ``width`` cells; the domain exterior counts as inside
    (mesh.py:130-141)."""
    out = mask.astype(bool, copy=True)
    for _ in range(width):
        h = out.copy()
        h[:, 1:] &= out[:, :-1]
        h[:, :-1] &= out[:, 1:]
        v = h.copy()
        v[1:, :] &= h[:-1, :]
        v[:-1, :] &= h[1:, :]
        out = v
    return out


def paint(boxes: np.ndarray, ny: int, nx: int) -> np.ndarray:
    """Boolean union of boxes over a (ny, nx) index space."""
    m = np.zeros((ny, nx), bool)
    for lo_i, lo_j, hi_i, hi_j in boxes:
        m[max(lo_j, 0):hi_j + 1, max(lo_i, 0):hi_i + 1] = True
    return m
