"""CPU checks of the measurement plumbing: the reference arm's JSON line on
a small configuration, the regrid-fill byte model, the native step tile
list."""

import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line_on_c2():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C2",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, MLAMR_REF_BUDGET_S="60"))
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    # the same workload string as the GPU arm's line
    assert d["config"]["workload"].startswith("C2: 2 levels, M=2, L1 128x128")
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_regrid_fill_bytes_model():
    from paper_1803_01450_b200.driver import regrid_fill_bytes
    M = 2
    new = np.array([[0, 0, 63, 63], [64, 0, 127, 63]])
    old = np.array([[0, 0, 63, 31]])
    refined = 2 * 64 * 64 - 64 * 32
    copied = 64 * 32
    want = 8 * (3 * M + 1 + (3 * M + 1) / 16) * refined + 8 * 6 * M * copied
    assert regrid_fill_bytes(new, old, 4, 4, M) == int(want)
    assert regrid_fill_bytes(new, np.zeros((0, 4)), 4, 4, M) == int(8 * (7 + 7 / 16) * 2 * 64 * 64)


def test_native_tile_list_matches_definition():
    from paper_1803_01450_b200.device import tile_list
    rng = np.random.default_rng(1)
    lo = rng.integers(0, 500, (300, 2))
    ext = rng.integers(1, 90, (300, 2))
    boxes = np.concatenate([lo, lo + ext - 1], axis=1)[:, [0, 1, 2, 3]].astype(np.int64)
    for shape in ((16, 32), (16, 16)):
        ty, tx = shape
        want = []
        for p, b in enumerate(boxes):
            nx, ny = b[2] - b[0] + 1, b[3] - b[1] + 1
            for a in range(-(-ny // ty)):
                for c in range(-(-nx // tx)):
                    want.append((p, a * ty, c * tx))
        assert np.array_equal(tile_list(boxes, shape), np.array(want, np.int32).reshape(-1, 3))
