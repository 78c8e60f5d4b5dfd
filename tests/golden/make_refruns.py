"""BASELINE configurations run by the REFERENCE itself (build container only:
imports ``mlamr`` from /root/reference/pkg/src, read-only) with the harness
plumbing of SURVEY.md App. B, so the configs are pinned to the reference and
not only to the oracle:

* a duck-typed ``Scenario`` serving the problem's seeded bathymetry and
  initial state (the methods used at src/regrid.py:83, :281, :287 and
  src/driver.py:115-117);
* a duck-typed ``RunConfig`` (src/driver.py:100-108) whose hierarchy is built
  from ``Hierarchy(domain, [LevelSpec...])`` directly, so C1's 256x4 strip
  with r = (4, 1) runs (src/mesh.py:345-351 rejects it; SURVEY probe 5);
* ``mlamr.regrid.flag_cells`` replaced by the harness gradient / Bernoulli
  rules where the problem uses them (called by module global, src/regrid.py:258);
* ``mlamr.regrid.cluster_flags`` wrapped with the harness max-patch chop
  (src/regrid.py:261);
* levels initialised by refinement where the harness does (C1's
  ``init_mode = "refine"``, C2's fixed 8x8 tiling): ``rebuild_child_level``
  with ``init_from_scenario=False`` at t = 0;
* the harness dynamic r_t (C5) as ``hier.levels[i] = replace(spec, r_t=...)``
  per coarse step;
* ``check_nesting=False`` (src/driver.py:97).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_refruns.py [C1 C2 C4r C5r]

Output ``tests/golden/ref_<name>.npz`` in the format of make_fullsize.py
(per-checkpoint layouts + per-patch interior digests, dts, r_t, counters,
mass), checked against the oracle (tests/test_oracle_refruns.py, CPU) and
the GPU (tests/test_gpu_fullsize.py).
"""

from __future__ import annotations

import os
import sys
import time
from dataclasses import replace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
for p in (REF, ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)

import mlamr.regrid as R  # noqa: E402
from mlamr import physics  # noqa: E402
from mlamr.driver import Simulation  # noqa: E402
from mlamr.errors import CflViolationError  # noqa: E402
from mlamr.mesh import Hierarchy, IndexBox, LevelSpec, dilate  # noqa: E402
from mlamr.regrid import RegridPolicy, rebuild_child_level  # noqa: E402
from mlamr.state import LayerParams, state_from_surfaces, surfaces_from_state  # noqa: E402

from make_fullsize import DIGEST_BYTES, patch_digest, ref_variant as variant  # noqa: E402

_ORIG_FLAG = R.flag_cells
_ORIG_CLUSTER = R.cluster_flags


class HarnessScenario:
    """Duck-typed mlamr.scenario.Scenario over a harness problem."""

    def __init__(self, pb):
        self.pb = pb

    def _box(self, patch):
        g = patch.ghost_width
        b = patch.box
        return (b.lo_i - g, b.lo_j - g, b.hi_i + g, b.hi_j + g)

    def fill_bathymetry(self, patch):
        patch.bathy[:, :] = self.pb.bathymetry_box(patch.level, self._box(patch))

    def rest_surfaces(self, bathy, params):
        # scenario.rest_surfaces (scenario.py:75-90) with the problem's rest levels
        eta = np.broadcast_to(np.asarray(self.pb.eta_rest, dtype=float).reshape((-1,) + (1,) * bathy.ndim),
                              (len(self.pb.eta_rest),) + bathy.shape)
        h, _ = state_from_surfaces(eta, bathy, params.dry_tolerance)
        return surfaces_from_state(h, bathy)

    def apply_initial_condition(self, patch, params):
        h, hu, hv = self.pb.initial_state_box(patch.level, self._box(patch))
        patch.h[...] = h
        patch.hu[...] = hu
        patch.hv[...] = hv
        patch.time = 0.0


class HarnessConfig:
    """Duck-typed mlamr.config.RunConfig (the members Simulation uses)."""

    def __init__(self, pb):
        self.pb = pb
        self.max_levels = pb.num_levels
        self.boundaries = dict(pb.boundaries)
        self.allowed_regions = tuple(pb.allowed_regions)
        self.cfl = pb.cfl
        self.dt_max = pb.dt_max

    def layer_params(self):
        pb = self.pb
        return LayerParams(num_layers=pb.num_layers, densities=tuple(pb.densities), gravity=pb.gravity,
                           dry_tolerance=pb.dry_tolerance)

    def scenario(self):
        return HarnessScenario(self.pb)

    def policy(self):
        pb = self.pb
        return RegridPolicy(wave_tolerance=tuple(pb.wave_tolerance), regrid_interval=pb.regrid_interval,
                            buffer_width=pb.buffer_width, efficiency_target=pb.efficiency_target)

    def build_hierarchy(self, uniform_fine=False):
        specs = [LevelSpec(*s) for s in self.pb.level_specs()]
        hier = Hierarchy(self.pb.domain, specs, self.pb.num_layers)
        hier.patches[1].append(hier.new_patch(1, hier.level_box(1)))
        return hier


class HarnessSimulation(Simulation):
    """mlamr.driver.Simulation with the harness initialisation by refinement
    (C1, C2) and the harness rules installed as module-global patches."""

    def __init__(self, pb):
        self.pb = pb
        self._fixed_init = None
        self._install()
        super().__init__(HarnessConfig(pb), workers=1, amr=True, check_nesting=False)

    def _install(self):
        pb = self.pb
        sim = self
        rule = pb.flag_rule

        def flag_cells(hier, level, policy, scenario, params):
            if rule[0] == "reference":
                return _ORIG_FLAG(hier, level, policy, scenario, params)
            s = hier.spec(level)
            covered = np.zeros((s.ny, s.nx), bool)
            for p in hier.patches[level]:
                covered[p.box.lo_j:p.box.hi_j + 1, p.box.lo_i:p.box.hi_i + 1] = True
            if rule[0] == "gradient":
                from paper_1803_01450_b200.problems import gradient_flags_map
                layers = list(rule[3])
                eta = np.zeros((len(layers), s.ny, s.nx))
                for p in hier.patches[level]:
                    jj, ii = p.interior
                    e = surfaces_from_state(p.h[:, jj, ii], p.bathy[jj, ii])
                    eta[:, p.box.lo_j:p.box.hi_j + 1, p.box.lo_i:p.box.hi_i + 1] = e[layers]
                f = gradient_flags_map(eta, covered, s.dx, s.dy, rule[1])
                return dilate(f, rule[2]) & covered
            if rule[0] == "bernoulli":
                f = pb.bernoulli_flags(level, sim.steps[level])
                return dilate(f, rule[2]) & covered
            raise ValueError(rule)

        def cluster_flags(flags, eff, allowed=None):
            if sim._fixed_init is not None:
                return sim._fixed_init
            boxes = _ORIG_CLUSTER(flags, eff, allowed)
            if pb.max_patch is None:
                return boxes
            from paper_1803_01450_b200.regrid import chop_boxes
            arr = np.array([(b.lo_i, b.lo_j, b.hi_i, b.hi_j) for b in boxes], np.int64).reshape(-1, 4)
            out = chop_boxes(arr, *pb.max_patch, aligned=pb.chop_aligned)
            return [IndexBox(*[int(v) for v in b]) for b in np.asarray(out).reshape(-1, 4)]

        R.flag_cells = flag_cells
        R.cluster_flags = cluster_flags

    def _rebuild(self, level, init_from_scenario=False):
        pb = self.pb
        fixed = pb.fixed_layout(level + 1) if init_from_scenario else None
        if init_from_scenario and (fixed is not None or pb.init_mode == "refine"):
            s = self.hier.spec(level)
            if fixed is not None:
                self._fixed_init = sorted((IndexBox(b[0] // s.r_x, b[1] // s.r_y, (b[2] + 1) // s.r_x - 1,
                                                    (b[3] + 1) // s.r_y - 1) for b in fixed),
                                          key=lambda b: (b.lo_j, b.lo_i))
            try:
                _, _, changed = rebuild_child_level(self.hier, level, self.policy, self.scenario, self.params,
                                                    self.cfg.boundaries, allowed_regions=self.cfg.allowed_regions,
                                                    init_from_scenario=False)
            finally:
                self._fixed_init = None
            return changed
        return super()._rebuild(level, init_from_scenario)

    # -- the harness coarse-step driver (driver.py:334-340 + App. B dynamic r_t)
    def choose_dt(self):
        dt = self.pb.dt_max
        for p in self.hier.patches[1]:
            dt = min(dt, physics.stable_dt(p, self.params, self.pb.cfl, self.pb.dt_max))
        return dt

    def apply_dynamic_rt(self, dt):
        if not self.pb.dynamic_rt:
            return
        dtl = dt
        for lev in range(1, self.hier.max_levels):
            s = self.hier.spec(lev)
            fs = self.hier.spec(lev + 1)
            sp = 0.0
            for p in self.hier.patches[lev + 1]:
                sp = max(sp, physics.observed_max_speed(p, self.params))
            rt = self.pb.pick_rt(sp, dtl, min(fs.dx, fs.dy), max(s.r_x, s.r_y))
            self.hier.levels[lev - 1] = replace(s, r_t=rt)
            dtl = dtl / rt


def checkpoint(sim, prefix, out):
    for lev, pats in sim.hier.patches.items():
        boxes = np.array([(p.box.lo_i, p.box.lo_j, p.box.hi_i, p.box.hi_j) for p in pats],
                         dtype=np.int32).reshape(-1, 4)
        dig = np.zeros((len(pats), DIGEST_BYTES), np.uint8)
        for k, p in enumerate(pats):
            jj, ii = p.interior
            dig[k] = np.frombuffer(patch_digest(p.h[:, jj, ii], p.hu[:, jj, ii], p.hv[:, jj, ii]), np.uint8)
        out[f"{prefix}L{lev}_boxes"] = boxes
        out[f"{prefix}L{lev}_digest"] = dig
    st = sim.stats
    out[f"{prefix}time"] = np.asarray(sim.time)
    out[f"{prefix}counters"] = np.array([st.total_cell_updates, st.num_regrids, st.hyperbolicity_warnings,
                                         st.wet_prefix_repairs], np.int64)
    out[f"{prefix}mass"] = np.asarray(sim.composite_mass())
    out[f"{prefix}rt"] = np.array([s.r_t for s in sim.hier.levels], np.int64)
    out[f"{prefix}sync_delta"] = np.asarray(st.sync_delta, float)
    out[f"{prefix}refine_delta"] = np.asarray(st.refine_delta, float)
    out[f"{prefix}derefine_delta"] = np.asarray(st.derefine_delta, float)
    out[f"{prefix}clipped"] = np.asarray(st.clipped_mass, float)


def run(name):
    pb, steps = variant(name)
    t0 = time.time()
    sim = HarnessSimulation(pb)
    out = {"name": np.asarray(name), "steps": np.asarray(steps), "source": np.asarray("reference")}
    checkpoint(sim, "s0_", out)
    print(f"[{name}] init {time.time() - t0:.1f} s, patches { {l: len(v) for l, v in sim.hier.patches.items()} }",
          flush=True)
    dts = []
    done = 0
    for k in range(1, steps + 1):
        dt = sim.choose_dt()
        sim.apply_dynamic_rt(dt)
        try:
            sim.advance_coarse_step(dt)
        except CflViolationError as exc:
            # the reference's own CFL guard fires (physics.py:342-347): the
            # fixture records where, and the GPU must raise it there too
            out["abort_step"] = np.asarray(k)
            out["abort_dt"] = np.asarray(dt)
            out["abort_rt"] = np.array([s.r_t for s in sim.hier.levels], np.int64)
            out["abort_msg"] = np.asarray(str(exc))
            print(f"[{name}] coarse step {k}: reference raised {exc}", flush=True)
            break
        dts.append(dt)
        done = k
        checkpoint(sim, f"s{k}_", out)
        print(f"[{name}] coarse step {k}: dt={dt!r} regrids {sim.stats.num_regrids} "
              f"patches { {l: len(v) for l, v in sim.hier.patches.items()} } ({time.time() - t0:.0f} s)",
              flush=True)
    out["dts"] = np.array(dts)
    out["done"] = np.asarray(done)
    path = os.path.join(HERE, f"ref_{name}.npz")
    np.savez_compressed(path, **out)
    R.flag_cells, R.cluster_flags = _ORIG_FLAG, _ORIG_CLUSTER
    return path


if __name__ == "__main__":
    for n in (sys.argv[1:] or ["C1", "C2", "C4r", "C5r"]):
        print("wrote", run(n), flush=True)
