"""Run configurations and the reference's scenario, as harness Problems.

``parse_config`` reads the reference's INI-style run files
(config.py:1-347 under /root/reference/pkg/src/mlamr): the same sections,
keys, defaults and validation, rejecting unknown sections/keys with a
``ConfigError`` that names the key.  ``problem_from_config`` turns the
result into a :class:`problems.Problem` carrying the reference's
``Scenario`` (scenario.py:22-123): flat or x-step beds sampled as exact
cell means at every level, and the rest state plus a right-moving pulse
with barotropic momenta as the initial condition.  Everything the GPU
driver needs then comes from the file, e.g.::

    from paper_1803_01450_b200.config import problem_from_config
    from paper_1803_01450_b200.driver import run_simulation
    pb = problem_from_config("configs/shelf_demo_small.cfg")
    run_simulation(pb, out_dir="out", t_final=pb.t_final, frame_times=pb.frame_times)

``tests/test_config.py`` checks the scenario fields bit for bit against the
arrays the reference's Scenario produced for shelf_demo_small, and
``tests/test_gpu_frames.py`` runs a config file to the reference's frames.
"""

from __future__ import annotations

import configparser
from dataclasses import dataclass, fields

import numpy as np

from .errors import ConfigError, MlamrError  # noqa: F401  (ConfigError re-exported)
from .problems import Problem


def _floats(text: str) -> tuple:
    return tuple(float(p) for p in (q.strip() for q in text.split(",")) if p)


def _ints(text: str) -> tuple:
    return tuple(int(p) for p in (q.strip() for q in text.split(",")) if p)


def _rects(text: str) -> tuple:
    out = []
    for chunk in (c.strip() for c in text.split(";")):
        if chunk:
            v = _floats(chunk)
            if len(v) != 4:
                raise ValueError(f"rectangle needs 4 values, got {chunk!r}")
            out.append(v)
    return tuple(out)


_REQ = object()
# section -> key -> (parser, default); the reference's schema (config.py:49-98)
SCHEMA = {
    "domain": {"x_min": (float, _REQ), "x_max": (float, _REQ), "y_min": (float, _REQ), "y_max": (float, _REQ)},
    "grid": {"nx": (int, _REQ), "ny": (int, _REQ), "max_levels": (int, 1), "refine_x": (_ints, ()),
             "refine_y": (_ints, ())},
    "time": {"t_final": (float, _REQ), "frame_times": (_floats, None), "cfl": (float, 0.9), "dt_max": (float, 1.0)},
    "physics": {"gravity": (float, 1.0), "num_layers": (int, 2), "density_ratio": (float, 0.95),
                "dry_tolerance": (float, 1e-3)},
    "scenario": {"name": (str, "unnamed"), "bathymetry": (str, _REQ), "b_level": (float, None),
                 "step_x": (float, None), "b_left": (float, None), "b_right": (float, None),
                 "eta_rest": (_floats, _REQ), "wave_amplitude": (float, 0.0), "wave_center": (float, 0.0),
                 "wave_width": (float, 1.0)},
    "boundaries": {"left": (str, "wall"), "right": (str, "wall"), "top": (str, "wall"), "bottom": (str, "wall")},
    "amr": {"wave_tolerance": (_floats, None), "regrid_interval": (int, 2), "buffer_width": (int, 2),
            "efficiency_target": (float, 0.7), "allowed_regions": (_rects, ())},
}
_DEFAULT_WAVE_TOL = (1e-2, 5e-2)


@dataclass
class RunConfig:
    """A resolved run file (field names as config.py:101-140)."""
    x_min: float
    x_max: float
    y_min: float
    y_max: float
    nx: int
    ny: int
    max_levels: int
    refine_x: tuple
    refine_y: tuple
    t_final: float
    frame_times: tuple
    cfl: float
    dt_max: float
    gravity: float
    num_layers: int
    density_ratio: float
    dry_tolerance: float
    name: str
    bathymetry: str
    b_level: float | None
    step_x: float | None
    b_left: float | None
    b_right: float | None
    eta_rest: tuple
    wave_amplitude: float
    wave_center: float
    wave_width: float
    left: str
    right: str
    top: str
    bottom: str
    wave_tolerance: tuple
    regrid_interval: int
    buffer_width: int
    efficiency_target: float
    allowed_regions: tuple

    @property
    def domain(self) -> tuple:
        return (self.x_min, self.x_max, self.y_min, self.y_max)

    @property
    def boundaries(self) -> dict:
        return {"left": self.left, "right": self.right, "top": self.top, "bottom": self.bottom}

    @property
    def densities(self) -> tuple:
        return (1.0,) if self.num_layers == 1 else (self.density_ratio, 1.0)

    def scenario(self) -> "Scenario":
        return Scenario(self.bathymetry, self.eta_rest, b_level=self.b_level, step_x=self.step_x,
                        b_left=self.b_left, b_right=self.b_right, wave_amplitude=self.wave_amplitude,
                        wave_center=self.wave_center, wave_width=self.wave_width, gravity=self.gravity)


def parse_config_text(text: str, source: str = "<text>") -> RunConfig:
    cp = configparser.ConfigParser(inline_comment_prefixes=("#",))
    cp.optionxform = str
    cp.read_string(text, source=source)
    return _resolve(cp)


def parse_config(path) -> RunConfig:
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise ConfigError(str(path), "config file not found") from None
    return parse_config_text(text, str(path))


def _resolve(cp: configparser.ConfigParser) -> RunConfig:
    for sec in cp.sections():
        if sec not in SCHEMA:
            raise ConfigError(sec, "unknown section")
        for key in cp[sec]:
            if key not in SCHEMA[sec]:
                raise ConfigError(f"{sec}.{key}", "unknown key")
    v = {}
    for sec, keys in SCHEMA.items():
        for key, (parse, default) in keys.items():
            if cp.has_option(sec, key):
                raw = cp.get(sec, key)
                try:
                    v[key] = parse(raw)
                except (TypeError, ValueError) as exc:
                    raise ConfigError(f"{sec}.{key}", f"cannot parse {raw!r}: {exc}") from None
            elif default is _REQ:
                raise ConfigError(f"{sec}.{key}", "required key missing")
            else:
                v[key] = default
    _validate(v)
    cfg = RunConfig(**{f.name: v[f.name] for f in fields(RunConfig)})
    try:
        cfg.scenario()
    except ValueError as exc:
        raise ConfigError("scenario", str(exc)) from None
    beds = [b for b in (cfg.b_level, cfg.b_left, cfg.b_right) if b is not None]
    if min(beds) >= cfg.eta_rest[-1]:
        raise ConfigError("scenario.eta_rest", "bathymetry must fall below the deepest rest surface somewhere")
    return cfg


def _validate(v: dict) -> None:
    """The reference's cross-checks (config.py:243-333)."""
    def need(ok, key, msg):
        if not ok:
            raise ConfigError(key, msg)

    need(v["x_max"] > v["x_min"], "domain.x_max", "domain width must be positive")
    need(v["y_max"] > v["y_min"], "domain.y_max", "domain height must be positive")
    need(v["nx"] >= 4 and v["ny"] >= 4, "grid.nx", "coarse grid must be at least 4x4")
    L = v["max_levels"]
    need(L >= 1, "grid.max_levels", "must be >= 1")
    for axis in ("refine_x", "refine_y"):
        need(L == 1 or len(v[axis]) == L - 1, f"grid.{axis}", f"need {L - 1} ratios for {L} levels")
        for r in v[axis]:
            need(r >= 2, f"grid.{axis}", f"refinement ratios must be >= 2, got {r}")
    if L == 1:
        v["refine_x"] = v["refine_y"] = ()
    need(v["t_final"] > 0, "time.t_final", "must be positive")
    need(0 < v["cfl"] <= 1, "time.cfl", "must be in (0, 1]")
    if v["frame_times"] is None:
        v["frame_times"] = (0.0, v["t_final"])
    ft = v["frame_times"]
    need(list(ft) == sorted(ft), "time.frame_times", "must be sorted")
    need(not ft or (ft[0] >= 0 and ft[-1] <= v["t_final"] + 1e-12), "time.frame_times",
         "must lie within [0, t_final]")
    need(v["num_layers"] in (1, 2), "physics.num_layers", "solver supports 1 or 2 layers")
    need(v["num_layers"] != 2 or 0 < v["density_ratio"] < 1, "physics.density_ratio", "must be in (0, 1)")
    need(v["dry_tolerance"] > 0, "physics.dry_tolerance", "must be positive")
    er = v["eta_rest"]
    need(len(er) == v["num_layers"], "scenario.eta_rest", "need one rest surface per layer")
    need(all(er[m] > er[m + 1] for m in range(len(er) - 1)), "scenario.eta_rest",
         "rest surfaces must strictly decrease with depth")
    need(v["wave_width"] > 0, "scenario.wave_width", "must be positive")
    for side in ("left", "right", "top", "bottom"):
        need(v[side] in ("wall", "outflow"), f"boundaries.{side}", "must be one of ('wall', 'outflow')")
    if v["wave_tolerance"] is None:
        v["wave_tolerance"] = _DEFAULT_WAVE_TOL[: v["num_layers"]]
    wt = v["wave_tolerance"]
    if len(wt) == 1 and v["num_layers"] > 1:
        v["wave_tolerance"] = wt = wt * v["num_layers"]
    need(len(wt) == v["num_layers"], "amr.wave_tolerance", "need one tolerance per layer (or a single value)")
    need(all(t > 0 for t in wt), "amr.wave_tolerance", "tolerances must be positive")
    need(v["regrid_interval"] >= 1, "amr.regrid_interval", "must be >= 1")
    need(v["buffer_width"] >= 0, "amr.buffer_width", "must be >= 0")
    need(0 < v["efficiency_target"] <= 1, "amr.efficiency_target", "must be in (0, 1]")


class Scenario:
    """Flat or x-step bed, layered rest surfaces and a Gaussian pulse on the
    free surface (scenario.py:22-123)."""

    def __init__(self, bathymetry, eta_rest, *, b_level=None, step_x=None, b_left=None, b_right=None,
                 wave_amplitude=0.0, wave_center=0.0, wave_width=1.0, gravity=1.0):
        if bathymetry not in ("flat", "step"):
            raise ValueError(f"unknown bathymetry kind {bathymetry!r}")
        if bathymetry == "flat" and b_level is None:
            raise ValueError("flat bathymetry needs b_level")
        if bathymetry == "step" and None in (step_x, b_left, b_right):
            raise ValueError("step bathymetry needs step_x, b_left, b_right")
        self.kind = bathymetry
        self.b_level, self.step_x, self.b_left, self.b_right = b_level, step_x, b_left, b_right
        self.eta_rest = tuple(float(e) for e in eta_rest)
        self.amp, self.center, self.width = wave_amplitude, wave_center, wave_width
        self.gravity = gravity

    def bed_means(self, x_lo: np.ndarray, x_hi: np.ndarray) -> np.ndarray:
        """Exact mean of the bed over [x_lo, x_hi] (scenario.py:56-65)."""
        x_lo = np.asarray(x_lo, dtype=float)
        x_hi = np.asarray(x_hi, dtype=float)
        if self.kind == "flat":
            return np.full_like(x_lo, self.b_level)
        w = x_hi - x_lo
        left = np.clip(self.step_x - x_lo, 0.0, w) / w
        return self.b_left * left + self.b_right * (1.0 - left)

    def pulse(self, x: np.ndarray) -> np.ndarray:
        x = np.asarray(x, dtype=float)
        if self.amp == 0.0:
            return np.zeros_like(x)
        a = (x - self.center) / self.width
        return self.amp * np.exp(-(a ** 2))

    def initial_state(self, xc: np.ndarray, B: np.ndarray, M: int, tol: float):
        """(h, hu, hv) over a box with bed B (scenario.py:96-123)."""
        ny = B.shape[0]
        pert = self.pulse(xc)[None, :] * np.ones((ny, 1))
        eta = np.broadcast_to(np.asarray(self.eta_rest).reshape(-1, 1, 1), (M,) + B.shape).copy()
        eta[0] = eta[0] + pert
        h = np.zeros_like(eta)
        bhat = np.zeros_like(eta[0]) + B
        for m in range(M - 1, -1, -1):
            h[m] = np.maximum(eta[m] - bhat, 0.0)
            bhat = bhat + h[m]
        rest = np.maximum(self.eta_rest[0] - B, 0.0)
        wet = rest > tol
        u = np.zeros_like(B)
        u[wet] = pert[wet] * np.sqrt(self.gravity / rest[wet])
        hu = h * u[None]
        hv = np.zeros_like(h)
        dry = h <= tol
        hu[dry] = 0.0
        hv[dry] = 0.0
        return h, hu, hv


def problem_from_config(cfg, uniform_fine: bool = False) -> Problem:
    """A Problem for the GPU driver from a RunConfig (or a path to a run
    file): geometry, layer parameters, regrid policy and allowed regions,
    frame times, and the scenario's per-level bed means and initial state.
    ``uniform_fine`` is the reference's ``--no-amr`` run (driver.py:104-107,
    config.py:191-206): one level at the finest level's resolution."""
    if not isinstance(cfg, RunConfig):
        cfg = parse_config(cfg)
    rx, ry = list(cfg.refine_x), list(cfg.refine_y)
    nx0, ny0 = cfg.nx, cfg.ny
    if uniform_fine and rx:
        for a, b in zip(rx, ry):
            nx0, ny0 = nx0 * a, ny0 * b
        rx, ry = [], []
    pb = Problem(
        name=cfg.name, domain=cfg.domain, coarse_nx=nx0, coarse_ny=ny0, ratios_x=rx, ratios_y=ry,
        ratios_t=[max(a, b) for a, b in zip(rx, ry)], num_layers=cfg.num_layers, densities=cfg.densities,
        gravity=cfg.gravity, dry_tolerance=cfg.dry_tolerance, eta_rest=cfg.eta_rest,
        boundaries=cfg.boundaries, cfl=cfg.cfl, dt_max=cfg.dt_max, wave_tolerance=tuple(cfg.wave_tolerance),
        regrid_interval=cfg.regrid_interval, buffer_width=cfg.buffer_width,
        efficiency_target=cfg.efficiency_target, flag_rule=("reference",), init_mode="scenario",
        notes=f"run file scenario {cfg.name!r}",
        allowed_regions=tuple(cfg.allowed_regions), t_final=cfg.t_final, frame_times=tuple(cfg.frame_times),
    )
    sc = cfg.scenario()
    x0 = cfg.x_min
    levels = []
    for (lev, nx, ny, dx, dy, *_r) in pb.level_specs():
        x = x0 + (np.arange(nx) + 0.5) * dx
        row = sc.bed_means(x - 0.5 * dx, x + 0.5 * dx)
        levels.append(np.ascontiguousarray(np.broadcast_to(row[None, :], (ny, nx))))
    pb.bathy_levels = levels
    M, tol = cfg.num_layers, cfg.dry_tolerance
    pb.ic = lambda p, level, xc, yc, jj, ii, B: sc.initial_state(xc, B, M, tol)
    pb.scenario = sc
    pb.amr_enabled = bool(rx)
    return pb
