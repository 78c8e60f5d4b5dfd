"""CPU checks of the C-ABI boundary: the library loads, exports every
entry point include/mlamr_b200.h declares, and its host-side native code
(clustering, regrid.py:129-182) matches the reference's golden vectors."""

import os
import re

import numpy as np

from conftest import ROOT, load_golden


def _declared():
    txt = open(os.path.join(ROOT, "include", "mlamr_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mlamr_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_1803_01450_b200 import _native
    L = _native.lib()
    names = _declared()
    assert len(names) >= 14
    for n in names:
        assert hasattr(L, n), n
        assert n in _native.SIGNATURES, n
    assert L.mlamr_version() >= 1
    assert b"sm_100a" in L.mlamr_build_info()


def test_native_cluster_flags_matches_reference_golden():
    from paper_1803_01450_b200.regrid import cluster_flags
    z = load_golden("cluster_cases.npz")
    for k in range(int(z["ncases"])):
        allowed = z[f"c{k}_allowed"]
        allowed = None if allowed.size == 0 else allowed
        boxes = cluster_flags(z[f"c{k}_flags"], float(z[f"c{k}_eff"]), allowed)
        got = np.array([list(b) for b in boxes], dtype=np.int64).reshape(-1, 4)
        assert np.array_equal(got, z[f"c{k}_boxes"]), k


def test_native_cluster_flags_matches_oracle_randomized(oracle):
    from paper_1803_01450_b200.mesh import dilate
    from paper_1803_01450_b200.regrid import cluster_flags
    rng = np.random.default_rng(7)
    for trial in range(60):
        ny, nx = int(rng.integers(1, 70)), int(rng.integers(1, 70))
        f = dilate(rng.random((ny, nx)) < rng.uniform(0.0, 0.2), int(rng.integers(0, 3)))
        eff = float(rng.choice([0.5, 0.7, 0.9, 1.0]))
        allowed = None
        if trial % 2:
            allowed = oracle.erode(rng.random((ny, nx)) > 0.05, 1)
            f &= allowed
        a = [tuple(b) for b in cluster_flags(f, eff, allowed)]
        b = [tuple(b) for b in oracle.cluster_flags(f, eff, allowed)]
        assert a == b, trial


def test_chop_and_nesting_host_logic(oracle):
    from paper_1803_01450_b200.mesh import IndexBox
    from paper_1803_01450_b200.regrid import chop, nesting_allowed
    boxes = [IndexBox(0, 0, 40, 17), IndexBox(50, 3, 52, 60)]
    for aligned in (False, True):
        got = [tuple(b) for b in chop(boxes, 16, 8, aligned)]
        ref = [tuple(b) for b in oracle.chop_boxes([oracle.Box(*b) for b in boxes], 16, 8, aligned)]
        assert got == ref
    rng = np.random.default_rng(3)
    bx = np.array([[2, 3, 20, 30], [25, 0, 40, 12]])
    m = nesting_allowed(bx, 32, 48)

    class P:
        def __init__(self, b):
            self.box = oracle.Box(*b)

    ref = oracle.nesting_allowed([P(b) for b in bx], oracle.Spec(1, 48, 32, 1.0, 1.0))
    assert np.array_equal(m, ref)
