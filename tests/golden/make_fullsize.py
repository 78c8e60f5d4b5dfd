"""Full-size parity fixtures: run the ORACLE (oracle/, pinned bit-exact to
the reference by tests/golden/make_golden.py + tests/test_oracle_golden.py)
on the BASELINE configurations at their full sizes and commit per-patch
digests of the interiors after each coarse step.

    python tests/golden/make_fullsize.py C4 [C3 C5 C5s ...] [--steps N]

The reference's own O(P^2) scans (ghost.py:186-196, regrid.py:311-323,
coarsen.py:46-75) cannot reach these sizes; the oracle restates them over a
bucket index (mlamr_oracle.BoxIndex) with unchanged order and arithmetic.

Output ``tests/golden/fullsize_<name>.npz`` (small): for every checkpoint
``s<k>_`` (after coarse step k; ``s0_`` = the initial hierarchy) the boxes of
every level (int32) and the first 8 bytes of one SHA-256 per patch of its interior ``h, hu, hv``
(float64, C order, +0.0 added so a zero's sign does not count -- the
parity tests compare bits up to the sign of zero), the coarse dt, the
per-level r_t, the run counters and the composite mass.
``tests/test_gpu_fullsize.py`` runs the GPU driver on the same problem and
compares.  Runs on CPU only (this container or any host); several minutes
to an hour per configuration.
"""

from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def problem(name: str):
    """The BASELINE problems at full size (problems.py); ``C5s`` is the
    regrid-stress variant of C5 (Bernoulli p = 0.05: the layout changes
    every coarse step, unlike p = 0.3 whose dilated flags cover ~96 % of
    the level and cluster to the same chopped layout every step)."""
    from paper_1803_01450_b200 import problems
    return problems.CONFIGS[name]()   # C5s: problems.config5_stress


def ref_variant(name: str):
    """(problem, coarse steps) of the configurations the REFERENCE itself
    runs (make_refruns.py): C1 and C2 at full size (C2 over its whole
    50-step schedule), C4 and C5 reduced to L1 64x64 (the reference's O(P^2)
    scans), with the regrid settings of the GPU parity variants
    (tests/test_gpu_driver.py)."""
    from paper_1803_01450_b200 import problems
    if name == "C1":
        return problems.config1(), 3
    if name == "C2":
        return problems.config2(), 50
    if name == "C4r":
        pb = problems.config4(nx0=64)
        pb.regrid_interval = 2
        return pb, 3
    if name == "C5r":
        pb = problems.config5(nx0=64)
        pb.bernoulli = (0.05,)
        pb.flag_rule = ("bernoulli", 0.05, 1)
        # the reference's CFL guard aborts coarse step 4 (Courant 1.193 on a
        # freshly refined level-2 patch): the fixture pins that abort too
        return pb, 4
    raise KeyError(name)


DIGEST_BYTES = 8


def patch_digest(h: np.ndarray, hu: np.ndarray, hv: np.ndarray) -> bytes:
    """SHA-256 of the interior fields (sign of zero canonicalised), first
    DIGEST_BYTES bytes: an equality check, not a security property."""
    d = hashlib.sha256()
    for a in (h, hu, hv):
        d.update(np.ascontiguousarray(a + 0.0, dtype="<f8").tobytes())
    return d.digest()[:DIGEST_BYTES]


def oracle_checkpoint(sim, prefix: str, out: dict) -> None:
    for lev, pats in sim.patches.items():
        boxes = np.array([tuple(p.box) for p in pats], dtype=np.int32).reshape(-1, 4)
        dig = np.zeros((len(pats), DIGEST_BYTES), np.uint8)
        for k, p in enumerate(pats):
            jj, ii = p.inner
            dig[k] = np.frombuffer(patch_digest(p.h[:, jj, ii], p.hu[:, jj, ii], p.hv[:, jj, ii]), np.uint8)
        out[f"{prefix}L{lev}_boxes"] = boxes
        out[f"{prefix}L{lev}_digest"] = dig
    st = sim.stats
    out[f"{prefix}time"] = np.asarray(sim.time)
    out[f"{prefix}counters"] = np.array([st.total_cell_updates, st.num_regrids, st.hyperbolicity_warnings,
                                         st.wet_prefix_repairs], np.int64)
    out[f"{prefix}mass"] = np.asarray(sim.composite_mass())
    out[f"{prefix}rt"] = np.array([s.r_t for s in sim.specs], np.int64)


def run(name: str, steps: int, workers: int) -> str:
    import mlamr_oracle as O
    O.build()
    pb = problem(name)
    t0 = time.time()
    sim = O.Simulation(pb, workers=workers)
    out = {"name": np.asarray(name), "steps": np.asarray(steps)}
    oracle_checkpoint(sim, "s0_", out)
    print(f"[{name}] init {time.time() - t0:.1f} s, patches "
          f"{ {l: len(v) for l, v in sim.patches.items()} }", flush=True)
    dts = []
    path = os.path.join(HERE, f"fullsize_{name}.npz")
    for k in range(1, steps + 1):
        t1 = time.time()
        dt = sim.choose_dt()
        sim.apply_dynamic_rt(dt)
        sim.advance_coarse_step(dt)
        dts.append(dt)
        oracle_checkpoint(sim, f"s{k}_", out)
        out["dts"] = np.array(dts)
        out["done"] = np.asarray(k)
        np.savez_compressed(path, **out)
        print(f"[{name}] coarse step {k}: dt={dt!r} {time.time() - t1:.1f} s, regrids "
              f"{sim.stats.num_regrids}, patches { {l: len(v) for l, v in sim.patches.items()} }",
              flush=True)
    return path


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--workers", type=int, default=2)
    a = ap.parse_args()
    for n in a.names:
        print("wrote", run(n, a.steps, a.workers), flush=True)


if __name__ == "__main__":
    main()
