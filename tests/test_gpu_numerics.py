"""The kernels' shared-reciprocal fp64 division must equal div.rn.f64 bit
for bit on every input (csrc/common.cuh: recip_nr / div_fast)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(a, b):
    import torch
    from paper_1803_01450_b200 import _native as N
    da = torch.from_numpy(a).cuda()
    db = torch.from_numpy(b).cuda()
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    slow = torch.zeros(1, dtype=torch.int64, device="cuda")
    N.check(N.lib().mlamr_selftest_div(da.data_ptr(), db.data_ptr(), len(a), bad.data_ptr(), slow.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream), "selftest_div")
    return int(bad.item()), int(slow.item())


def test_div_fast_equals_ieee_division_random():
    rng = np.random.default_rng(11)
    n = 1 << 24
    for scale in (1.0, 1e-3, 1e3, 1e-150, 1e150):
        a = rng.standard_normal(n) * np.exp(rng.uniform(-20, 20, n)) * scale
        b = rng.standard_normal(n) * np.exp(rng.uniform(-20, 20, n))
        bad, slow = _run(a, b)
        assert bad == 0, (scale, bad)
    # raw random bit patterns: every exponent, NaN/inf/denormals included
    a = rng.integers(0, 2 ** 63, n, dtype=np.int64).view(np.float64) * np.where(rng.random(n) < 0.5, -1, 1)
    b = rng.integers(0, 2 ** 63, n, dtype=np.int64).view(np.float64)
    bad, slow = _run(a, b)
    assert bad == 0 and slow > 0


def test_div_fast_special_values():
    vals = np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 2.2250738585072014e-308,
                     1.7976931348623157e308, 1e-300, 1e300, 3.0, 0.1, 1e-3, 9.81])
    a, b = np.meshgrid(vals, vals)
    bad, slow = _run(a.ravel().copy(), b.ravel().copy())
    assert bad == 0


def test_div_fast_zero_dividend():
    # +-0 over normal finite divisors of every magnitude: signed zero, exact
    rng = np.random.default_rng(12)
    n = 1 << 20
    b = rng.standard_normal(n) * np.exp(rng.uniform(-700, 700, n))
    b = b[np.isfinite(b) & (np.abs(b) >= 2.2250738585072014e-308)]
    a = np.where(rng.random(len(b)) < 0.5, 0.0, -0.0)
    bad, slow = _run(a, b.copy())
    assert bad == 0
