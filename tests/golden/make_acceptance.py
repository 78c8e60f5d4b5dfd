"""Golden vectors for the reference's two refine/coarsen acceptance cases,
produced by running the REFERENCE itself (build container only: imports
``mlamr`` from /root/reference/pkg/src, read-only).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_acceptance.py

The cases restate the setup of /root/reference/pkg/tests/test_acceptance.py:
``_telescoping_pair`` (:109-126) -- a 16x8 level 1 on (0,4)x(0,1), r=2,
one fine patch IndexBox(8, 4, 23, 11) with seeded bathymetry whose coarse
values are its exact block means, a fully wet seeded coarse state --
followed by

* ``coarsen-refine-identity`` (:145-165), seeds 100-104: refine_patch then
  average_down; the reference FAILS its own 1e-13 tolerance here
  (acceptance_report.txt:4, worst 2.84e-01), a behaviour the GPU path must
  reproduce rather than fix;
* ``conditional-mass-conservation`` (:129-142), seeds 0-4: block means of
  the refined depths equal the coarse depths (worst 1.67e-15).

Per case the fixture stores the inputs (coarse arrays with ghosts, fine
bathymetry), the reference's refined fine arrays, its coarse arrays after
average_down, and the worst deviations the acceptance test computes.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF)

from mlamr.coarsen import average_down, block_mean  # noqa: E402
from mlamr.mesh import IndexBox, build_hierarchy  # noqa: E402
from mlamr.refine import coarse_data_from_patch, refine_patch  # noqa: E402
from mlamr.state import LayerParams  # noqa: E402


def _pair(seed):
    # test_acceptance.py:109-126, restated (same calls, same draw order)
    hier = build_hierarchy((0.0, 4.0, 0.0, 1.0), 16, 8, [2], [2], num_layers=2)
    coarse = hier.patches[1][0]
    fine = hier.new_patch(2, IndexBox(8, 4, 23, 11))
    rng = np.random.default_rng(seed)
    fjj, fii = fine.interior
    fine.bathy[:, :] = -6.0
    fine.bathy[fjj, fii] = rng.uniform(-6.0, -5.0, (fine.box.ny, fine.box.nx))
    cb = fine.box.coarsened(2, 2)
    jj, ii = coarse.local_slices(cb)
    coarse.bathy[:, :] = -5.5
    coarse.bathy[jj, ii] = block_mean(fine.bathy[fjj, fii], 2, 2)
    coarse.h[:, :, :] = rng.uniform(0.5, 1.5, coarse.h.shape)
    coarse.hu[:, :, :] = rng.uniform(-0.2, 0.2, coarse.hu.shape)
    coarse.hv[:, :, :] = rng.uniform(-0.2, 0.2, coarse.hv.shape)
    return coarse, fine, (jj, ii), (fjj, fii)


def main():
    params = LayerParams(2, (0.95, 1.0), gravity=1.0, dry_tolerance=1e-3)
    rec = {}
    worst_id = 0.0
    worst_cons = 0.0
    k = 0
    for kind, seeds in (("identity", range(100, 105)), ("conservation", range(5))):
        for seed in seeds:
            coarse, fine, (jj, ii), (fjj, fii) = _pair(seed)
            pre = {f"c{k}_in_{f}": getattr(coarse, f).copy() for f in ("h", "hu", "hv", "bathy")}
            rec.update(pre)
            rec[f"c{k}_fine_bathy"] = fine.bathy.copy()
            rec[f"c{k}_kind"] = np.array(kind)
            rec[f"c{k}_seed"] = np.array(seed)
            # the fine patch's ghost frame is never written by refine_patch
            # (region = interior); record its pre-refine contents too
            for f in ("h", "hu", "hv"):
                rec[f"c{k}_fine_pre_{f}"] = getattr(fine, f).copy()
            refine_patch(coarse_data_from_patch(coarse), fine, 2, 2, params)
            for f in ("h", "hu", "hv"):
                rec[f"c{k}_fine_{f}"] = getattr(fine, f).copy()
            if kind == "identity":
                before = (coarse.h[:, jj, ii].copy(), coarse.hu[:, jj, ii].copy(), coarse.hv[:, jj, ii].copy())
                average_down([fine], [coarse], 2, 2, params)
                for f in ("h", "hu", "hv"):
                    rec[f"c{k}_coarse_{f}"] = getattr(coarse, f).copy()
                after = (coarse.h[:, jj, ii], coarse.hu[:, jj, ii], coarse.hv[:, jj, ii])
                w = 0.0
                for b, a in zip(before, after):
                    scale = np.maximum(np.abs(b), 1e-3)
                    w = max(w, float((np.abs(a - b) / scale).max()))
                rec[f"c{k}_worst"] = np.array(w)
                worst_id = max(worst_id, w)
            else:
                means = block_mean(fine.h[:, fjj, fii], 2, 2)
                rel = np.abs(means - coarse.h[:, jj, ii]) / np.abs(coarse.h[:, jj, ii])
                w = float(rel.max())
                rec[f"c{k}_worst"] = np.array(w)
                worst_cons = max(worst_cons, w)
            k += 1
    rec["ncases"] = np.array(k)
    rec["worst_identity"] = np.array(worst_id)
    rec["worst_conservation"] = np.array(worst_cons)
    path = os.path.join(OUT, "acceptance_cases.npz")
    np.savez_compressed(path, **rec)
    print("wrote", path, "worst identity %.3g, worst conservation %.3g" % (worst_id, worst_cons))


if __name__ == "__main__":
    main()
