"""Generate golden vectors by running the REFERENCE itself (build container
only: it imports ``mlamr`` from /root/reference/pkg/src, read-only).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Outputs (committed, small): tests/golden/*.npz.  Every fixture stores the
seeded inputs and the reference's outputs; the oracle and the GPU path are
checked against them (tests/test_oracle_golden.py, tests/test_gpu_*.py).
Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF)

from mlamr import coarsen, ghost, physics, refine, regrid  # noqa: E402
from mlamr.config import parse_config  # noqa: E402
from mlamr.driver import Simulation  # noqa: E402
from mlamr.errors import CflViolationError  # noqa: E402
from mlamr.mesh import IndexBox, build_hierarchy  # noqa: E402
from mlamr.refine import CoarseData  # noqa: E402
from mlamr.state import LayerParams  # noqa: E402

WALLS = {"left": "wall", "right": "wall", "top": "wall", "bottom": "wall"}
MIXED = {"left": "outflow", "right": "wall", "top": "wall", "bottom": "outflow"}


def _save(name, **arrays):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays)
    print("wrote", path, sum(a.nbytes for a in arrays.values()), "bytes raw")


def _random_state(rng, M, NY, NX, kind):
    """Seeded two/one-layer states with dry cells, thin layers and fronts."""
    B = -1.0 + 0.6 * rng.random((NY, NX))
    if kind == "front":
        B[:, NX // 2:] += 0.7
    eta_top = 0.05 * rng.standard_normal((NY, NX))
    if M == 1:
        h = np.maximum(eta_top - B, 0.0)[None]
    else:
        eta_if = -0.5 + 0.05 * rng.standard_normal((NY, NX))
        h1 = np.maximum(eta_if - B, 0.0)
        h0 = np.maximum(eta_top - (B + h1), 0.0)
        h = np.stack([h0, h1])
        if kind == "prefix":
            # water under a dry layer: forces the wet-prefix repair
            mask = rng.random((NY, NX)) < 0.2
            mask[: NY // 2, : NX // 2] = True
            h[0][mask] = 0.0
    hu = 0.3 * rng.standard_normal((M, NY, NX)) * h
    hv = 0.3 * rng.standard_normal((M, NY, NX)) * h
    if kind == "shear" and M == 2:
        hu[0] += 2.0 * h[0]
        hu[1] -= 2.0 * h[1]
    return B, h, hu, hv


def make_step_cases(rng):
    """physics.step_patch (physics.py:330-386) on seeded patches, several
    consecutive steps with wall/outflow BCs between them."""
    recs = {}
    k = 0
    for M in (1, 2):
        for kind in ("plain", "front", "prefix", "shear"):
            for (nx, ny) in ((7, 5), (12, 9), (16, 16)):
                hier = build_hierarchy((0.0, 1.0 * nx / ny, 0.0, 1.0), nx, ny, [], [], num_layers=M)
                p = hier.patches[1][0]
                B, h, hu, hv = _random_state(rng, M, ny + 4, nx + 4, kind)
                p.bathy[...] = B
                p.h[...] = h
                p.hu[...] = hu
                p.hv[...] = hv
                dens = (1.0,) if M == 1 else (0.95, 1.0)
                prm = LayerParams(M, dens, gravity=1.0, dry_tolerance=1e-3)
                bcs = WALLS if k % 2 == 0 else MIXED
                ghost.apply_bathymetry_bcs(p, bcs, hier.level_box(1))
                rec = {"M": M, "nx": nx, "ny": ny, "bcs": 0 if bcs is WALLS else 1,
                       "dx": p.dx, "dy": p.dy, "B": p.bathy.copy()}
                ghost.apply_state_bcs(p, bcs, hier.level_box(1))
                rec["h0"], rec["hu0"], rec["hv0"] = p.h.copy(), p.hu.copy(), p.hv.copy()
                outs = []
                for s in range(4):
                    if s > 0:
                        ghost.apply_state_bcs(p, bcs, hier.level_box(1))
                    dt = physics.stable_dt(p, prm, 0.6)
                    yf = bool(s % 2)
                    pre = (p.h.copy(), p.hu.copy(), p.hv.copy())
                    r = physics.step_patch(p, dt, prm, y_first=yf)
                    outs.append((dt, yf, pre, (p.h.copy(), p.hu.copy(), p.hv.copy()), r))
                for s, (dt, yf, pre, post, r) in enumerate(outs):
                    rec[f"s{s}_dt"] = dt
                    rec[f"s{s}_yfirst"] = int(yf)
                    rec[f"s{s}_pre_h"], rec[f"s{s}_pre_hu"], rec[f"s{s}_pre_hv"] = pre
                    rec[f"s{s}_h"], rec[f"s{s}_hu"], rec[f"s{s}_hv"] = post
                    rec[f"s{s}_speed"] = r.max_wave_speed
                    rec[f"s{s}_fixes"] = r.hyperbolicity_fixes
                    rec[f"s{s}_repairs"] = r.wet_prefix_repairs
                    rec[f"s{s}_clipped"] = np.asarray(r.clipped_mass)
                    rec[f"s{s}_mass_delta"] = np.asarray(r.mass_delta)
                for key, v in rec.items():
                    recs[f"c{k}_{key}"] = np.asarray(v)
                k += 1
    # CFL violation case (physics.py:342-347): raised before any update
    hier = build_hierarchy((0.0, 1.0, 0.0, 1.0), 8, 8, [], [], num_layers=2)
    p = hier.patches[1][0]
    B, h, hu, hv = _random_state(rng, 2, 12, 12, "plain")
    p.bathy[...] = B
    p.h[...] = h
    p.hu[...] = hu
    p.hv[...] = hv
    prm = LayerParams(2, (0.95, 1.0), gravity=1.0, dry_tolerance=1e-3)
    dt = 3.0 * physics.stable_dt(p, prm, 1.0)
    try:
        physics.step_patch(p, dt, prm)
        raised = 0
    except CflViolationError:
        raised = 1
    recs["cfl_B"], recs["cfl_h"], recs["cfl_hu"], recs["cfl_hv"] = B, h, hu, hv
    recs["cfl_dt"] = np.asarray(dt)
    recs["cfl_raised"] = np.asarray(raised)
    recs["ncases"] = np.asarray(k)
    _save("step_cases.npz", **recs)


def make_interp_cases(rng):
    """refine.interpolate_state (refine.py:158-190) on seeded gathered data
    with unavailable cells and dry layers."""
    recs = {}
    k = 0
    for M in (1, 2, 3):
        for (rx, ry) in ((2, 2), (4, 4), (4, 2), (2, 4), (4, 1)):
            for trial in range(3):
                cnx, cny = int(rng.integers(3, 8)), int(rng.integers(3, 8))
                clo = (int(rng.integers(-2, 5)), int(rng.integers(-2, 5)))
                cbox = IndexBox(clo[0], clo[1], clo[0] + cnx - 1, clo[1] + cny - 1)
                B = -1.0 + 0.8 * rng.random((cny, cnx))
                eta = np.sort(0.1 * rng.standard_normal((M, cny, cnx)) - np.arange(M)[:, None, None] * 0.3, axis=0)[::-1]
                from mlamr.state import state_from_surfaces
                h, _ = state_from_surfaces(eta, B, 1e-3)
                hu = rng.standard_normal((M, cny, cnx)) * h
                hv = rng.standard_normal((M, cny, cnx)) * h
                avail = rng.random((cny, cnx)) > 0.15
                h[:, ~avail] = 0.0
                hu[:, ~avail] = 0.0
                hv[:, ~avail] = 0.0
                B[~avail] = 0.0
                cd = CoarseData(cbox, h, hu, hv, B, avail)
                # fine box: parents strictly inside the coarse box
                pi0 = cbox.lo_i + 1
                pj0 = cbox.lo_j + 1
                pi1 = cbox.hi_i - 1 if cnx > 2 else cbox.hi_i
                pj1 = cbox.hi_j - 1 if cny > 2 else cbox.hi_j
                fi0 = pi0 * rx + int(rng.integers(0, rx))
                fj0 = pj0 * ry + int(rng.integers(0, ry))
                fi1 = max(fi0, (pi1 + 1) * rx - 1 - int(rng.integers(0, rx)))
                fj1 = max(fj0, (pj1 + 1) * ry - 1 - int(rng.integers(0, ry)))
                fbox = IndexBox(fi0, fj0, fi1, fj1)
                fb = -1.0 + 0.8 * rng.random((fbox.ny, fbox.nx))
                dens = tuple(np.linspace(0.9, 1.0, M)) if M > 1 else (1.0,)
                prm = LayerParams(M, dens, gravity=1.0, dry_tolerance=1e-3)
                oh, ohu, ohv = refine.interpolate_state(cd, fbox, fb, rx, ry, prm)
                rec = dict(M=M, rx=rx, ry=ry, cbox=np.array(cbox[:] if False else [cbox.lo_i, cbox.lo_j, cbox.hi_i, cbox.hi_j]),
                           fbox=np.array([fbox.lo_i, fbox.lo_j, fbox.hi_i, fbox.hi_j]),
                           h=h, hu=hu, hv=hv, B=B, avail=avail, fb=fb, oh=oh, ohu=ohu, ohv=ohv)
                for key, v in rec.items():
                    recs[f"c{k}_{key}"] = np.asarray(v)
                k += 1
    recs["ncases"] = np.asarray(k)
    _save("interp_cases.npz", **recs)


def make_blockmean_cases(rng):
    recs = {}
    k = 0
    for (rx, ry) in ((2, 2), (4, 4), (4, 2), (2, 4), (4, 1), (1, 4), (2, 1)):
        a = rng.standard_normal((2, ry * 5, rx * 7)) * rng.uniform(0, 1e3, (2, ry * 5, rx * 7))
        recs[f"c{k}_a"] = a
        recs[f"c{k}_r"] = np.array([rx, ry])
        recs[f"c{k}_out"] = coarsen.block_mean(a, rx, ry)
        k += 1
    # patches ONE coarse cell wide (numpy then sums each r_y x r_x block as
    # one contiguous pairwise run) and one coarse cell tall, in a strided
    # view like average_down's fp.h[:, fjj, fii] (coarsen.py:59); own rng so
    # the fixtures generated after this one keep their inputs
    nr = np.random.default_rng(1803)
    for (rx, ry) in ((2, 2), (4, 4), (4, 2), (2, 4), (4, 1), (2, 1)):
        for (cny, cnx) in ((5, 1), (1, 1), (1, 6), (3, 2)):
            big = nr.standard_normal((2, ry * cny + 4, rx * cnx + 4)) * nr.uniform(0, 1e3, (2, ry * cny + 4, rx * cnx + 4))
            a = big[:, 2:-2, 2:-2]
            recs[f"c{k}_a"] = np.ascontiguousarray(a)
            recs[f"c{k}_r"] = np.array([rx, ry])
            recs[f"c{k}_out"] = coarsen.block_mean(a, rx, ry)
            k += 1
    recs["ncases"] = np.asarray(k)
    _save("blockmean_cases.npz", **recs)


def make_cluster_cases(rng):
    """regrid.cluster_flags (regrid.py:129-182) on seeded flag maps."""
    from mlamr.mesh import dilate, erode
    recs = {}
    k = 0
    for (ny, nx, p, dil) in ((16, 24, 0.05, 1), (32, 32, 0.02, 2), (40, 64, 0.01, 2),
                              (24, 24, 0.3, 1), (64, 48, 0.004, 3), (20, 20, 0.0, 0)):
        for eff in (0.7, 0.9):
            f = dilate(rng.random((ny, nx)) < p, dil)
            allowed = erode(rng.random((ny, nx)) > 0.02, 1) if k % 3 == 1 else None
            if allowed is not None:
                f &= allowed
            boxes = regrid.cluster_flags(f, eff, allowed)
            recs[f"c{k}_flags"] = f
            recs[f"c{k}_allowed"] = allowed if allowed is not None else np.ones((0, 0), bool)
            recs[f"c{k}_eff"] = np.asarray(eff)
            recs[f"c{k}_boxes"] = np.array([[b.lo_i, b.lo_j, b.hi_i, b.hi_j] for b in boxes],
                                           dtype=np.int64).reshape(-1, 4)
            k += 1
    m = rng.random((30, 30)) < 0.5
    recs["dilate_in"] = m
    recs["dilate_out"] = dilate(m, 2)
    recs["erode_out"] = erode(m, 1)
    recs["ncases"] = np.asarray(k)
    _save("cluster_cases.npz", **recs)


def _level_arrays(cfg, sim):
    """Per-level reference scenario data over each full level box plus the
    2-cell frame (scenario.py:68-125), for the oracle/GPU adapter problem."""
    out = {}
    hier = sim.hier
    for s in hier.levels:
        p = hier.new_patch(s.level, hier.level_box(s.level))
        sim.scenario.fill_bathymetry(p)
        sim.scenario.apply_initial_condition(p, sim.params)
        out[f"L{s.level}_bathy"] = p.bathy.copy()
        out[f"L{s.level}_h"] = p.h.copy()
        out[f"L{s.level}_hu"] = p.hu.copy()
        out[f"L{s.level}_hv"] = p.hv.copy()
        out[f"L{s.level}_spec"] = np.array([s.nx, s.ny, s.r_x, s.r_y, s.r_t])
        out[f"L{s.level}_dxdy"] = np.array([s.dx, s.dy])
    return out


def _dump_hier(prefix, hier):
    out = {}
    for lev, plist in hier.patches.items():
        out[f"{prefix}L{lev}_boxes"] = np.array(
            [[p.box.lo_i, p.box.lo_j, p.box.hi_i, p.box.hi_j] for p in plist], dtype=np.int64
        ).reshape(-1, 4)
        for k, p in enumerate(plist):
            out[f"{prefix}L{lev}_p{k}_h"] = p.h.copy()
            out[f"{prefix}L{lev}_p{k}_hu"] = p.hu.copy()
            out[f"{prefix}L{lev}_p{k}_hv"] = p.hv.copy()
            out[f"{prefix}L{lev}_p{k}_bathy"] = p.bathy.copy()
    return out


def make_run_cases():
    """driver.Simulation on configs/shelf_demo_small.cfg (3 levels, r=2,2):
    the t=0 hierarchy, then fixed coarse steps with the reference's own
    regrid/fill/step/coarsen; also one isolated level-ghost fill with a
    time-blended parent (driver.py:157-190)."""
    cfg = parse_config("/root/reference/pkg/configs/shelf_demo_small.cfg")
    sim = Simulation(cfg, workers=1)
    recs = _level_arrays(cfg, sim)
    recs.update(_dump_hier("t0_", sim.hier))
    recs["cfl"] = np.asarray(cfg.cfl)
    recs["dt_max"] = np.asarray(cfg.dt_max)
    dts = []
    nsteps = 4
    for step in range(nsteps):
        dt = cfg.dt_max
        for p in sim.hier.patches[1]:
            dt = min(dt, physics.stable_dt(p, sim.params, cfg.cfl, cfg.dt_max))
        dts.append(dt)
        sim.advance_coarse_step(dt)
        if step == 1:
            recs.update(_dump_hier("s2_", sim.hier))
    recs.update(_dump_hier("final_", sim.hier))
    recs["dts"] = np.array(dts)
    st = sim.stats
    recs["stat_total_cell_updates"] = np.asarray(st.total_cell_updates)
    recs["stat_num_regrids"] = np.asarray(st.num_regrids)
    recs["stat_fixes"] = np.asarray(st.hyperbolicity_warnings)
    recs["stat_repairs"] = np.asarray(st.wet_prefix_repairs)
    recs["stat_clipped"] = np.asarray(st.clipped_mass)
    recs["stat_refine_delta"] = np.asarray(st.refine_delta)
    recs["stat_derefine_delta"] = np.asarray(st.derefine_delta)
    recs["stat_sync_delta"] = np.asarray(st.sync_delta)
    recs["stat_initial_mass"] = np.asarray(st.initial_mass)
    recs["final_mass"] = np.asarray(sim.composite_mass())
    recs["steps"] = np.array([sim.steps[l] for l in sorted(sim.steps)])

    # isolated ghost fill of level 3 with a blended level-2 parent
    lev = 3
    parents = sim.hier.patches[lev - 1]
    t0 = sim.hier.patches[lev - 1][0].time
    old = {id(p): (p.h * 0.999, p.hu * 1.001, p.hv * 0.998) for p in parents}
    sim._stash[lev - 1] = (t0 - 0.01, 0.01, old)
    for p in parents:
        recs_key = f"gf_parent_{parents.index(p)}"
        recs[recs_key + "_oh"], recs[recs_key + "_ohu"], recs[recs_key + "_ohv"] = old[id(p)]
    before = _dump_hier("gf_before_", sim.hier)
    sim.fill_level_ghosts(lev, t0 - 0.0037)
    after = _dump_hier("gf_after_", sim.hier)
    recs.update(before)
    recs.update(after)
    recs["gf_t"] = np.asarray(t0 - 0.0037)
    recs["gf_t0"] = np.asarray(t0 - 0.01)
    recs["gf_dt"] = np.asarray(0.01)
    _save("run_shelf_small.npz", **recs)


def make_frame_cases():
    """Frames the reference itself writes (frames.frame_from_hierarchy +
    write_frame) for configs/shelf_demo_small.cfg at t=0 and after two
    coarse steps, binary and text; the t=0 text frame must equal the
    reference's committed fixture tests/fixtures/frames/shelf_small_frame0000.txt."""
    import io
    import tempfile
    from mlamr import frames as F
    cfg = parse_config("/root/reference/pkg/configs/shelf_demo_small.cfg")
    sim = Simulation(cfg, workers=1)
    recs = {}

    def grab(tag):
        fr = F.frame_from_hierarchy(sim.hier, sim.time, cfg.eta_rest)
        for text in (False, True):
            with tempfile.NamedTemporaryFile(suffix=".frame") as tf:
                F.write_frame(fr, tf.name, text_mode=text)
                recs[f"{tag}_{'txt' if text else 'bin'}"] = np.frombuffer(open(tf.name, "rb").read(), np.uint8)

    grab("t0")
    fixture = "/root/reference/pkg/tests/fixtures/frames/shelf_small_frame0000.txt"
    assert recs["t0_txt"].tobytes() == open(fixture, "rb").read(), "t0 text frame differs from the fixture"
    dts = []
    for _ in range(2):
        dt = cfg.dt_max
        for p in sim.hier.patches[1]:
            dt = min(dt, physics.stable_dt(p, sim.params, cfg.cfl, cfg.dt_max))
        dts.append(dt)
        sim.advance_coarse_step(dt)
    grab("s2")
    recs["dts"] = np.array(dts)
    # the full run_simulation (driver.py:365-410) to t_final with its frame
    # times: frame files and stats.json
    import json
    from mlamr.driver import run_simulation
    with tempfile.TemporaryDirectory() as d:
        run_simulation(cfg, out_dir=d, workers=1)
        for k in range(len(cfg.frame_times)):
            recs[f"run_frame{k}"] = np.frombuffer(open(os.path.join(d, f"frame{k:04d}.bin"), "rb").read(), np.uint8)
        st = json.load(open(os.path.join(d, "stats.json")))
    for key in ("wall_time", "cpu_time"):
        st.pop(key)
    recs["run_stats_json"] = np.frombuffer(json.dumps(st, sort_keys=True).encode(), np.uint8)
    # the uniform-grid run (--no-amr, driver.py:104-107) at the finest resolution
    with tempfile.TemporaryDirectory() as d:
        run_simulation(cfg, out_dir=d, workers=1, amr=False)
        recs["uniform_frame_last"] = np.frombuffer(
            open(os.path.join(d, f"frame{len(cfg.frame_times) - 1:04d}.bin"), "rb").read(), np.uint8)
        st = json.load(open(os.path.join(d, "stats.json")))
    for key in ("wall_time", "cpu_time"):
        st.pop(key)
    recs["uniform_stats_json"] = np.frombuffer(json.dumps(st, sort_keys=True).encode(), np.uint8)
    recs["run_t_final"] = np.asarray(cfg.t_final)
    recs["run_frame_times"] = np.asarray(cfg.frame_times)
    _save("frames_shelf_small.npz", **recs)


def main():
    rng = np.random.default_rng(20180305)
    make_step_cases(rng)
    make_interp_cases(rng)
    make_blockmean_cases(rng)
    make_cluster_cases(rng)
    make_run_cases()
    make_frame_cases()


if __name__ == "__main__":
    main()
