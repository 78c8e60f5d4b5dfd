"""Shared driver for the digest fixtures (tests/golden/make_fullsize.py,
tests/golden/make_refruns.py): run a simulation (the oracle or the GPU
driver) along a fixture's coarse steps and compare every checkpoint."""

import os
import sys

import numpy as np

from conftest import GOLDEN

if GOLDEN not in sys.path:
    sys.path.insert(0, GOLDEN)

from make_fullsize import DIGEST_BYTES, patch_digest  # noqa: E402


def digest_arrays(items):
    """items: iterable of (h, hu, hv) interiors -> [n, DIGEST_BYTES] uint8."""
    rows = [np.frombuffer(patch_digest(h, hu, hv), np.uint8) for (h, hu, hv) in items]
    return np.stack(rows) if rows else np.zeros((0, DIGEST_BYTES), np.uint8)


def oracle_levels(sim):
    out = {}
    for lev, pats in sim.patches.items():
        boxes = np.array([tuple(p.box) for p in pats], np.int32).reshape(-1, 4)
        items = []
        for p in pats:
            jj, ii = p.inner
            items.append((p.h[:, jj, ii], p.hu[:, jj, ii], p.hv[:, jj, ii]))
        out[lev] = (boxes, digest_arrays(items))
    return out


def gpu_levels(sim):
    out = {}
    g = 2
    for lev, pool in sim.levels.items():
        host = pool.download()
        items = []
        for p in range(pool.P):
            h, hu, hv, _ = pool.patch_arrays(p, host=host)
            items.append((h[:, g:-g, g:-g], hu[:, g:-g, g:-g], hv[:, g:-g, g:-g]))
        out[lev] = (pool.boxes.astype(np.int32), digest_arrays(items))
    return out


def check(z, prefix, levels, counters, mass, rt, stats=None):
    """levels: {lev: (boxes, digests)}; counters: [updates, regrids, fixes,
    repairs]; stats: RunStats-like with the mass diagnostics (optional)."""
    bad = []
    for lev, (boxes, dig) in sorted(levels.items()):
        key = f"{prefix}L{lev}_boxes"
        if key not in z:
            assert len(boxes) == 0, (prefix, lev)
            continue
        assert np.array_equal(boxes, z[key]), f"{prefix} level {lev}: layout differs"
        diff = np.flatnonzero((dig != z[f"{prefix}L{lev}_digest"]).any(axis=1))
        if len(diff):
            bad.append((lev, len(diff), diff[:5].tolist(), len(dig)))
    assert not bad, f"{prefix}: patches whose interiors differ (level, count, first, of): {bad}"
    assert [int(c) for c in counters] == z[f"{prefix}counters"].tolist(), (prefix, counters)
    ref_mass = z[f"{prefix}mass"]
    np.testing.assert_allclose(mass, ref_mass, rtol=1e-12)
    assert [int(r) for r in rt] == z[f"{prefix}rt"].tolist(), (prefix, rt)
    if stats is not None and f"{prefix}sync_delta" in z:
        # mass diagnostics: sums in another order (numpy pairwise vs tree
        # reductions) of ~1e14 m^3 terms, compared at 1e-11 of the mass scale
        scale = float(np.abs(ref_mass).sum())
        for name, mine in (("sync_delta", stats.sync_delta), ("refine_delta", stats.refine_delta),
                           ("derefine_delta", stats.derefine_delta), ("clipped", stats.clipped_mass)):
            ref = z[f"{prefix}{name}"]
            got = np.asarray(mine if len(mine) else np.zeros(len(ref)), float)
            np.testing.assert_allclose(got, ref, rtol=0, atol=1e-11 * scale, err_msg=f"{prefix}{name}")


def fixture(name):
    path = os.path.join(GOLDEN, name)
    return np.load(path) if os.path.exists(path) else None
