"""Seeded synthetic inputs for the BASELINE configurations C1-C5.

The reference ships no datasets for these configurations and its
``Scenario`` (scenario.py:22-123 under /root/reference/pkg/src/mlamr) can
only express flat or x-step beds, so every configuration here is a harness
problem in the sense of SURVEY.md App. B: geometry, layer parameters, an
analytic bathymetry sampled at finest-level cell centres and block-averaged
upward (so the ladder telescopes exactly, coarsen.py:79-100), analytic
initial surfaces, and the harness rules the reference lacks (gradient and
Bernoulli flag rules, a max-patch-size chop, dynamic r_t, fixed initial
layouts).

Everything is generated on the host with numpy from one master seed per
configuration; the GPU path and the CPU oracle consume the same arrays
byte for byte.  Per-cell random values use a counter-based hash of the
global cell index, so any sub-box evaluates identically whatever the patch
layout.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from math import prod
from typing import Callable, Optional

import numpy as np

WALLS = {"left": "wall", "right": "wall", "bottom": "wall", "top": "wall"}


# ---------------------------------------------------------------------------
# counter-based uniforms (splitmix64 finaliser over the global cell index)
# ---------------------------------------------------------------------------
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_GOLD = np.uint64(0x9E3779B97F4A7C15)


def hash_uniform(seed: int, stream: int, jj: np.ndarray, ii: np.ndarray) -> np.ndarray:
    """Uniform [0,1) per (seed, stream, j, i); layout-independent."""
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) * _GOLD + np.uint64(stream) * _M2
             + (jj.astype(np.int64).astype(np.uint64) << np.uint64(32))
             + ii.astype(np.int64).astype(np.uint64))
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def state_from_surfaces(eta: np.ndarray, bathy: np.ndarray) -> np.ndarray:
    """Depths from surfaces, bottom layer first (state.py:72-101)."""
    M = eta.shape[0]
    h = np.zeros_like(eta)
    bhat = np.zeros_like(eta[0]) + bathy
    for m in range(M - 1, -1, -1):
        h[m] = np.maximum(eta[m] - bhat, 0.0)
        bhat = bhat + h[m]
    return h


def block_mean(a: np.ndarray, rx: int, ry: int) -> np.ndarray:
    """numpy block mean, the same expression the reference evaluates
    (coarsen.py:21-27), so coarse bathymetry telescopes bit-exactly."""
    ny, nx = a.shape[-2], a.shape[-1]
    return a.reshape(a.shape[:-2] + (ny // ry, ry, nx // rx, rx)).mean(axis=(-3, -1))


# ---------------------------------------------------------------------------
# problem description
# ---------------------------------------------------------------------------
@dataclass
class Problem:
    """A harness problem: everything both the GPU path and the oracle need."""

    name: str
    domain: tuple
    coarse_nx: int
    coarse_ny: int
    ratios_x: list
    ratios_y: list
    ratios_t: list
    num_layers: int
    densities: tuple
    gravity: float
    dry_tolerance: float
    eta_rest: tuple
    boundaries: dict = field(default_factory=lambda: dict(WALLS))
    cfl: float = 0.7
    dt_max: float = 1.0e9
    wave_tolerance: tuple = (0.1, 0.1)
    regrid_interval: int = 2
    buffer_width: int = 2
    efficiency_target: float = 0.7
    flag_rule: tuple = ("reference",)
    max_patch: Optional[tuple] = None
    chop_aligned: bool = False       # cut at global multiples of max_patch
    dynamic_rt: bool = False
    n_coarse_steps: int = 10
    seed: int = 0
    # per-level in-domain bathymetry (level 1 first)
    bathy_levels: list = field(default_factory=list)
    # initial state evaluator: (problem, level, xc[nx], yc[ny], jj, ii, B) -> (h, hu, hv)
    ic: Optional[Callable] = None
    fixed_layouts: dict = field(default_factory=dict)
    bernoulli: Optional[tuple] = None  # (p,)
    # how levels >= 2 get data at t=0: "scenario" (the initial condition,
    # regrid.py:284-286) or "refine" (interpolated from the level below)
    init_mode: str = "scenario"
    # physical rectangles (x0, x1, y0, y1) refinement is confined to, by a
    # cell-centre test (regrid.nesting_allowed, regrid.py:185-211)
    allowed_regions: tuple = ()
    # run length and frame times of a run file (config.py); 0 / () = unset
    t_final: float = 0.0
    frame_times: tuple = ()
    notes: str = ""

    def region_mask(self, level: int) -> Optional[np.ndarray]:
        """Cells of ``level`` whose centre lies in an allowed region (None
        when no regions are configured)."""
        if not self.allowed_regions:
            return None
        lev, nx, ny, dx, dy = self.level_specs()[level - 1][:5]
        xc = self.domain[0] + (np.arange(nx) + 0.5) * dx
        yc = self.domain[2] + (np.arange(ny) + 0.5) * dy
        inside = np.zeros((ny, nx), bool)
        for x0, x1, y0, y1 in self.allowed_regions:
            inside |= (xc[None, :] >= x0) & (xc[None, :] <= x1) & (yc[:, None] >= y0) & (yc[:, None] <= y1)
        return inside

    # -- geometry (mesh.py:325-375) -----------------------------------------
    def level_specs(self):
        x0, x1, y0, y1 = self.domain
        w, hgt = x1 - x0, y1 - y0
        L = len(self.ratios_x) + 1
        out = []
        for lev in range(1, L + 1):
            nx = self.coarse_nx * prod(self.ratios_x[: lev - 1])
            ny = self.coarse_ny * prod(self.ratios_y[: lev - 1])
            if lev <= len(self.ratios_x):
                rx, ry, rt = self.ratios_x[lev - 1], self.ratios_y[lev - 1], self.ratios_t[lev - 1]
            else:
                rx = ry = rt = 1
            out.append((lev, nx, ny, w / nx, h_div(hgt, ny), rx, ry, rt))
        return out

    @property
    def num_levels(self) -> int:
        return len(self.ratios_x) + 1

    def cell_centers(self, level: int, box) -> tuple:
        lev, nx, ny, dx, dy = self.level_specs()[level - 1][:5]
        ii = np.arange(box[0], box[2] + 1)
        jj = np.arange(box[1], box[3] + 1)
        return self.domain[0] + (ii + 0.5) * dx, self.domain[2] + (jj + 0.5) * dy, jj, ii

    def bathymetry_box(self, level: int, box) -> np.ndarray:
        """In-domain cells from the level array; out-of-domain cells are 0
        (the caller's boundary conditions overwrite them, ghost.py:118-129)."""
        lo_i, lo_j, hi_i, hi_j = box
        B = self.bathy_levels[level - 1]
        ny, nx = B.shape
        out = np.zeros((hi_j - lo_j + 1, hi_i - lo_i + 1))
        a_i, a_j = max(lo_i, 0), max(lo_j, 0)
        b_i, b_j = min(hi_i, nx - 1), min(hi_j, ny - 1)
        if a_i <= b_i and a_j <= b_j:
            out[a_j - lo_j:b_j - lo_j + 1, a_i - lo_i:b_i - lo_i + 1] = B[a_j:b_j + 1, a_i:b_i + 1]
        return out

    def initial_state_box(self, level: int, box):
        xc, yc, jj, ii = self.cell_centers(level, box)
        B = self.bathymetry_box(level, box)
        return self.ic(self, level, xc, yc, jj, ii, B)

    def fixed_layout(self, level: int):
        return self.fixed_layouts.get(level)

    # -- harness rules --------------------------------------
    def pick_rt(self, speed: float, dt_level: float, dmin_fine: float, rmax: int) -> int:
        """Dynamic r_t: smallest r_t in [1, rmax] with
        speed * (dt_level / r_t) / dmin_fine <= cfl."""
        for rt in range(1, rmax + 1):
            if speed * (dt_level / rt) / dmin_fine <= self.cfl:
                return rt
        return rmax

    def bernoulli_flags(self, level: int, step: int) -> np.ndarray:
        """Flags re-seeded every regrid: Bernoulli(p) per coarse cell,
        counter-hashed on (seed, level, step, j, i)."""
        lev, nx, ny = self.level_specs()[level - 1][:3]
        jj, ii = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
        u = hash_uniform(self.seed, 1000 + 97 * level + 7919 * step, jj, ii)
        return u < self.bernoulli[0]


def h_div(a: float, n: int) -> float:
    return a / n


def gradient_flags_map(eta: np.ndarray, covered: np.ndarray, dx: float, dy: float,
                       tol: float) -> np.ndarray:
    """Harness gradient rule (C1, C3): a covered cell is flagged when the
    surface difference across any face shared with another covered cell,
    divided by the cell size, exceeds ``tol`` in magnitude.  ``eta`` is
    [K, ny, nx] (the surfaces tested); layout-independent."""
    f = np.zeros(covered.shape, bool)
    for k in range(eta.shape[0]):
        e = eta[k]
        gx = np.abs(e[:, 1:] - e[:, :-1]) / dx > tol
        gx &= covered[:, 1:] & covered[:, :-1]
        gy = np.abs(e[1:, :] - e[:-1, :]) / dy > tol
        gy &= covered[1:, :] & covered[:-1, :]
        f[:, 1:] |= gx
        f[:, :-1] |= gx
        f[1:, :] |= gy
        f[:-1, :] |= gy
    return f & covered


# ---------------------------------------------------------------------------
# field building blocks
# ---------------------------------------------------------------------------
def _finest_bathymetry(pb: Problem, fn: Callable[[np.ndarray, np.ndarray], np.ndarray],
                       rows_per_chunk: int = 512) -> None:
    """Sample B at finest-level centres, then block-mean upward."""
    specs = pb.level_specs()
    lev, nx, ny, dx, dy = specs[-1][:5]
    x = pb.domain[0] + (np.arange(nx) + 0.5) * dx
    Bf = np.empty((ny, nx))
    for j0 in range(0, ny, rows_per_chunk):
        j1 = min(ny, j0 + rows_per_chunk)
        y = pb.domain[2] + (np.arange(j0, j1) + 0.5) * dy
        Bf[j0:j1] = fn(x[None, :], y[:, None])
    levels = [Bf]
    for k in range(len(specs) - 2, -1, -1):
        rx, ry = specs[k][5], specs[k][6]
        levels.append(block_mean(levels[-1], rx, ry))
    pb.bathy_levels = levels[::-1]


def _gaussian_sum(x, y, bumps):
    """Sum of isotropic Gaussians evaluated as separable outer products
    (x a row vector, y a column vector)."""
    out = np.zeros(np.broadcast(x, y).shape)
    for (a, cx, cy, w) in bumps:
        out = out + (a * np.exp(-((y - cy) / w) ** 2)) * np.exp(-((x - cx) / w) ** 2)
    return out


def _windowed_bumps(B, x, y, bumps, nsig=6.0):
    """Add Gaussian bumps only within nsig widths of their centre (the
    definition of the harness bathymetry; exact outside is irrelevant)."""
    xs = x.ravel()
    ys = y.ravel()
    for (a, cx, cy, w) in bumps:
        i0 = np.searchsorted(xs, cx - nsig * w)
        i1 = np.searchsorted(xs, cx + nsig * w)
        j0 = np.searchsorted(ys, cy - nsig * w)
        j1 = np.searchsorted(ys, cy + nsig * w)
        if i0 >= i1 or j0 >= j1:
            continue
        xx = xs[i0:i1][None, :]
        yy = ys[j0:j1][:, None]
        B[j0:j1, i0:i1] = B[j0:j1, i0:i1] + a * np.exp(-(((xx - cx) / w) ** 2 + ((yy - cy) / w) ** 2))
    return B


def _fourier_noise(rng, K: int, sigma: float, L: float, kmax: int = 6):
    ax = rng.integers(-kmax, kmax + 1, size=K)
    ay = rng.integers(1, kmax + 1, size=K)
    ph = rng.uniform(0, 2 * np.pi, size=K)
    c = rng.standard_normal(K) * sigma * np.sqrt(2.0 / K)
    return list(zip(ax, ay, ph, c, [L] * K))


def _eval_noise(x, y, modes):
    """Sum of plane waves c*cos(kx x + ky y + ph), separably:
    cos(a + b) = cos a cos b - sin a sin b (x row vector, y column)."""
    out = np.zeros(np.broadcast(x, y).shape)
    for (ax, ay, ph, c, L) in modes:
        a = 2 * np.pi * ax * x / L
        b = 2 * np.pi * ay * y / L + ph
        out = out + ((c * np.cos(b)) * np.cos(a) - (c * np.sin(b)) * np.sin(a))
    return out


# ---------------------------------------------------------------------------
# C1: 1-D two-layer strip
# ---------------------------------------------------------------------------
def config1(seed: int = 1, n_coarse_steps: int = 3) -> Problem:
    nx = 256
    dx = 1.0e5 / nx
    pb = Problem(
        name="C1", domain=(0.0, 1.0e5, 0.0, 4 * dx), coarse_nx=nx, coarse_ny=4,
        ratios_x=[4], ratios_y=[1], ratios_t=[4], num_layers=2,
        densities=(0.97, 1.0), gravity=9.81, dry_tolerance=1e-3,
        eta_rest=(0.0, -200.0), cfl=0.7, wave_tolerance=(1e-2, 1e-1),
        regrid_interval=10**9, buffer_width=2, flag_rule=("gradient", 1e-5, 2, (0,)),
        n_coarse_steps=n_coarse_steps, seed=seed,
        notes="1 refine at t=0 (gradient flags |d eta_1/dx| > 1e-5), then coarse steps",
    )
    _finest_bathymetry(pb, lambda x, y: -4000.0 + 4050.0 * x / 1.0e5 + 0.0 * y)

    def ic(p, level, xc, yc, jj, ii, B):
        X = xc[None, :] + 0.0 * yc[:, None]
        e1 = 0.5 * np.exp(-(((X - 5.0e4) / 5.0e3) ** 2))
        e2 = -200.0 + 2.0 * np.exp(-(((X - 4.0e4) / 8.0e3) ** 2))
        h = state_from_surfaces(np.stack([e1, e2]), B)
        return h, np.zeros_like(h), np.zeros_like(h)

    pb.ic = ic
    pb.init_mode = "refine"
    return pb


# ---------------------------------------------------------------------------
# C2 / C4 family: parabolic basin with bumps, Gaussian surface, noisy interface
# ---------------------------------------------------------------------------
def _basin_problem(name, seed, nx0, L, levels_r, nbumps, pulse, n_coarse_steps,
                   regrid_interval, max_patch, wave_tol, fixed_layouts=None, dynamic_rt=False,
                   ratios_y=None, bernoulli=None, flag_rule=("reference",)) -> Problem:
    rng = np.random.default_rng(seed)
    rx = list(levels_r)
    ry = list(ratios_y if ratios_y is not None else levels_r)
    pb = Problem(
        name=name, domain=(0.0, L, 0.0, L), coarse_nx=nx0, coarse_ny=nx0,
        ratios_x=rx, ratios_y=ry, ratios_t=[max(a, b) for a, b in zip(rx, ry)],
        num_layers=2, densities=(0.97, 1.0), gravity=9.81, dry_tolerance=1e-3,
        eta_rest=(0.0, -150.0), cfl=0.7, wave_tolerance=wave_tol,
        regrid_interval=regrid_interval, buffer_width=2, max_patch=max_patch,
        n_coarse_steps=n_coarse_steps, seed=seed, dynamic_rt=dynamic_rt,
        bernoulli=bernoulli, flag_rule=flag_rule,
    )
    s = L / 2.0e5
    c = L / 2.0
    bumps = [(rng.uniform(-200, 200), rng.uniform(0, L), rng.uniform(0, L),
              rng.uniform(5e3, 2e4) * s) for _ in range(nbumps)]
    R = L / 2.0

    def bed(x, y):
        r2 = (x - c) ** 2 + (y - c) ** 2
        return -3000.0 + 3100.0 * (r2 / (R * R))

    def bed_full(x, y):
        # dry land is capped flat at +10 m: refinement interpolates surfaces
        # against the finer bed (refine.py:175-189), so steep dry terrain
        # would sprout thin puddles wherever a fine bed lies below its
        # coarse mean, and their thin-film velocities trip the CFL guard
        B = bed(x, y) + _gaussian_sum(x, y, bumps)
        return np.minimum(B, 10.0)

    _finest_bathymetry(pb, bed_full)
    surf = [(rng.uniform(0.2, 1.0), rng.uniform(0.25 * L, 0.75 * L), rng.uniform(0.25 * L, 0.75 * L),
             rng.uniform(1.0e4, 3.0e4) * s) for _ in range(4)]
    noise = _fourier_noise(rng, 12, 0.5, L)
    pulse_c = (0.3 * L, 0.5 * L)
    g = pb.gravity

    def ic(p, level, xc, yc, jj, ii, B):
        X = xc[None, :]
        Y = yc[:, None]
        e1 = _gaussian_sum(X, Y, surf)
        pert = None
        if pulse:
            pert = 1.0 * np.exp(-(((X - pulse_c[0]) / 2.0e4) ** 2 + ((Y - pulse_c[1]) / 2.0e4) ** 2))
            e1 = e1 + pert
        e2 = -150.0 + _eval_noise(X, Y, noise)
        h = state_from_surfaces(np.stack([np.broadcast_to(e1, B.shape), np.broadcast_to(e2, B.shape)]), B)
        JJ, II = np.meshgrid(jj, ii, indexing="ij")
        hu = np.empty_like(h)
        hv = np.empty_like(h)
        # momenta U[-0.1,0.1]*h, tapered to zero in layers thinner than 50 m:
        # refinement interpolates momenta independently of depth
        # (refine.py:182-186), so momentum next to a wet/dry front would
        # otherwise become huge velocities in thin fine cells
        taper = np.clip((h - 50.0) / 100.0, 0.0, 1.0)
        for m in range(2):
            hu[m] = (0.2 * hash_uniform(p.seed, 10 * level + 2 * m, JJ, II) - 0.1) * h[m] * taper[m]
            hv[m] = (0.2 * hash_uniform(p.seed, 10 * level + 2 * m + 1, JJ, II) - 0.1) * h[m] * taper[m]
        if pert is not None:
            total = np.maximum(0.0 - B, 0.0)
            wet = total > p.dry_tolerance
            u = np.zeros_like(B)
            pb_ = np.broadcast_to(pert, B.shape)
            u[wet] = pb_[wet] * np.sqrt(g / total[wet])
            for m in range(2):
                hu[m] = hu[m] + h[m] * u * taper[m]
        dry = h <= p.dry_tolerance
        hu[dry] = 0.0
        hv[dry] = 0.0
        return h, hu, hv

    pb.ic = ic
    pb.fixed_layouts = fixed_layouts or {}
    return pb


def config2(seed: int = 2, n_coarse_steps: int = 50) -> Problem:
    """C2: L1 128x128 on [0,2e5]^2, r=4, 64 level-2 patches of 32x32 tiling
    the centre at t=0 (initialised by refinement), regrid every 5 with the
    reference rule and a 32x32 (fine) chop."""
    boxes = [(128 + 32 * a, 128 + 32 * b, 128 + 32 * a + 31, 128 + 32 * b + 31)
             for b in range(8) for a in range(8)]
    return _basin_problem("C2", seed, 128, 2.0e5, [4], 8, False, n_coarse_steps, 5, (8, 8),
                          (0.05, 0.6), fixed_layouts={2: boxes})



def config4(seed: int = 4, n_coarse_steps: int = 200, nx0: int = 512) -> Problem:
    """C4: L1 512x512 on [0,1e6]^2, r=4,4, ~8192 level-3 patches of 64x64
    from the reference rule + a 64x64 chop, regrid every 10.

    dry_tolerance = 1 cm: with the reference's 1 mm the pulse's run-up
    leaves millimetre films on the beach whose momenta give |u| ~ 300 m/s,
    and the reference's own CFL guard aborts the run near coarse step 31
    (at cfl 0.7, 0.45 and 0.3 alike, tools/c4_variants.py).  With 1 cm the
    full 200-step schedule completes with level-3 speeds <= 171 m/s."""
    pb = _basin_problem("C4", seed, nx0, 1.0e6 * nx0 / 512, [4, 4], 64, True, n_coarse_steps,
                        10, (16, 16), (0.1, 0.6))
    pb.chop_aligned = True
    pb.dry_tolerance = 1.0e-2
    return pb


def config5(seed: int = 5, n_coarse_steps: int = 100, nx0: int = 1280) -> Problem:
    """C5: L1 1280x1280, r=(4,2), dynamic r_t, Bernoulli(0.3) flags per L1
    cell re-seeded every step, dilated by 1, clustered, chopped to 16x16
    fine patches (4x8 coarse)."""
    return _basin_problem("C5", seed, nx0, 1.25e3 * nx0, [4], 16, False, n_coarse_steps, 1,
                          (4, 8), (0.05, 0.6), dynamic_rt=True, ratios_y=[2],
                          bernoulli=(0.3,), flag_rule=("bernoulli", 0.3, 1))


# ---------------------------------------------------------------------------
# C3: three layers over a continental shelf
# ---------------------------------------------------------------------------
def config3(seed: int = 3, n_coarse_steps: int = 100, nx0: int = 256) -> Problem:
    """C3.  cfl = 0.5: at 0.7 the three-layer model (the M=3 generalisation
    the reference rejects) blows up in its fourth coarse step in freshly
    refined level-3 patches at the x = 0 edge, in the CPU oracle exactly as
    on the GPU and at every size tried (nx0 = 32..256); at 0.5 the full-size
    run completes its 100 coarse steps (tools/full_runs.py)."""
    rng = np.random.default_rng(seed)
    L = 4.0e5 * nx0 / 256
    r1, r2 = 0.97, 0.985
    pb = Problem(
        name="C3", domain=(0.0, L, 0.0, L), coarse_nx=nx0, coarse_ny=nx0,
        ratios_x=[4, 4], ratios_y=[4, 4], ratios_t=[4, 4], num_layers=3,
        densities=(r1 * r2, r2, 1.0), gravity=9.81, dry_tolerance=1e-3,
        eta_rest=(0.0, -100.0, -600.0), cfl=0.5, wave_tolerance=(0.1, 1.0, 1.0),
        regrid_interval=10, buffer_width=2, max_patch=(16, 16),
        flag_rule=("gradient", 2.0e-4, 2, (1, 2)), dynamic_rt=True,
        n_coarse_steps=n_coarse_steps, seed=seed,
    )
    bumps = [(rng.uniform(100, 600), rng.uniform(0.3 * L, 0.9 * L), rng.uniform(0, L),
              rng.uniform(5e3, 2e4)) for _ in range(24)]

    def bed(x, y):
        B = -4000.0 + 4020.0 * (x / L) + 0.0 * y
        return np.minimum(_windowed_bumps(B, x, y, bumps), 20.0)

    _finest_bathymetry(pb, bed)
    n1 = _fourier_noise(rng, 10, 5.0 / 2.0, L)
    n2 = _fourier_noise(rng, 10, 5.0 / 2.0, L)

    def ic(p, level, xc, yc, jj, ii, B):
        X = xc[None, :]
        Y = yc[:, None]
        e0 = np.zeros(B.shape)
        e1 = np.broadcast_to(-100.0 + np.clip(_eval_noise(X, Y, n1), -5, 5), B.shape)
        e2 = np.broadcast_to(-600.0 + np.clip(_eval_noise(X, Y, n2), -5, 5), B.shape)
        h = state_from_surfaces(np.stack([e0, e1, e2]), B)
        return h, np.zeros_like(h), np.zeros_like(h)

    pb.ic = ic
    return pb


def config5_stress(seed: int = 5, n_coarse_steps: int = 100, nx0: int = 1280, p: float = 0.05) -> Problem:
    """C5 as a regrid stress that actually regrids: with Bernoulli(0.3)
    flags dilated by one cell nearly every level-1 cell is flagged, the
    clustered layout is the same every step and C5 performs no rebuild at
    all (profiles/r01/README.md); at p = 0.05 the dilated flags cover ~37 %
    of level 1 and the level-2 layout (~75 k 16x16 patches) is rebuilt --
    refine, copy, derefine -- in every coarse step.  Its dynamic-r_t rule
    (pick_rt, from the speeds before the rebuild) meets the reference's CFL
    guard in the fourth coarse step (t = 19.17): freshly refined patches are
    faster than the ones r_t was chosen for."""
    pb = config5(seed, n_coarse_steps, nx0)
    pb.name = "C5s"
    pb.bernoulli = (p,)
    pb.flag_rule = ("bernoulli", p, 1)
    return pb


CONFIGS = {"C1": config1, "C2": config2, "C3": config3, "C4": config4, "C5": config5, "C5s": config5_stress}
