"""Parity at the BASELINE sizes: the GPU driver on full-size C3, C4 (the
bench configuration), C5 and the C5 regrid-stress variant, against
per-patch digests of the oracle's interiors after every coarse step
(tests/golden/make_fullsize.py; the oracle is pinned bit-exact to the
reference by tests/test_oracle_golden.py).

Layouts must be identical, every patch's (h, hu, hv) interior bit-identical
(sign of zero aside), the coarse dt and per-level r_t identical, the
counters equal and the composite mass within 1e-12 relative (its sums are
ordered differently).  Size-only faults -- int32 index arithmetic, plan
offsets, chop fragments at 16k-75k patches -- show up here and nowhere
else."""

import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu
sys.path.insert(0, GOLDEN)

NAMES = ["C3", "C4", "C5", "C5s"]


def _digests(sim, level):
    from make_fullsize import DIGEST_BYTES, patch_digest
    pool = sim.levels[level]
    host = pool.download()
    boxes = pool.boxes.astype(np.int32)
    dig = np.zeros((pool.P, DIGEST_BYTES), np.uint8)
    g = 2
    for p in range(pool.P):
        h, hu, hv, _ = pool.patch_arrays(p, host=host)
        dig[p] = np.frombuffer(patch_digest(h[:, g:-g, g:-g], hu[:, g:-g, g:-g], hv[:, g:-g, g:-g]), np.uint8)
    return boxes, dig


def _check(sim, z, prefix):
    bad = []
    for lev in range(1, sim.L + 1):
        boxes, dig = _digests(sim, lev)
        assert np.array_equal(boxes, z[f"{prefix}L{lev}_boxes"]), f"{prefix} level {lev}: layout differs"
        diff = np.flatnonzero((dig != z[f"{prefix}L{lev}_digest"]).any(axis=1))
        if len(diff):
            bad.append((lev, len(diff), diff[:5].tolist(), len(dig)))
    assert not bad, f"{prefix}: patches whose interiors differ (level, count, first, of): {bad}"
    st = sim.finish()
    got = [st.total_cell_updates, st.num_regrids, st.hyperbolicity_warnings, st.wet_prefix_repairs]
    assert got == z[f"{prefix}counters"].tolist(), (prefix, got)
    np.testing.assert_allclose(sim.composite_mass(), z[f"{prefix}mass"], rtol=1e-12)


@pytest.mark.parametrize("name", NAMES)
def test_full_size_matches_oracle(name):
    path = os.path.join(GOLDEN, f"fullsize_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    from make_fullsize import problem
    from paper_1803_01450_b200.driver import Simulation
    z = np.load(path)
    pb = problem(name)
    sim = Simulation(pb)
    _check(sim, z, "s0_")
    for k in range(1, int(z["done"]) + 1):
        dt = sim.choose_dt()
        assert dt == float(z["dts"][k - 1]), (k, dt, float(z["dts"][k - 1]))
        sim.apply_dynamic_rt(dt)
        assert [s.r_t for s in sim.specs] == z[f"s{k}_rt"].tolist()
        sim.advance_coarse_step(dt)
        assert sim.time == float(z[f"s{k}_time"])
        _check(sim, z, f"s{k}_")
    sim.close()
