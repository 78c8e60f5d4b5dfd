"""Parity of whole runs against digest fixtures, on the GPU:

* the BASELINE configurations at FULL size -- C3, C4 (the bench
  configuration), C5 and the C5 regrid-stress variant -- against the oracle
  (tests/golden/make_fullsize.py; the oracle is pinned bit-exact to the
  reference by tests/test_oracle_golden.py and tests/test_oracle_refruns.py);
* C1, C2 (full size, C2's whole 50-step schedule), C4 and C5 (reduced)
  against the REFERENCE's own runs (tests/golden/make_refruns.py), C5's
  ending in the reference's CFL abort.

Layouts identical, every patch's (h, hu, hv) interior bit-identical (sign of
zero aside), coarse dt and per-level r_t identical, counters equal, the
composite mass within 1e-12 relative and the reference runs' mass
diagnostics (sync / refine / derefine delta, clipped mass) within 1e-11 of
the mass scale.  Size-only faults -- int32 index arithmetic, plan offsets,
chop fragments at 16k-75k patches -- show up here and nowhere else."""

import numpy as np
import pytest

from fixture_runs import check, fixture, gpu_levels

pytestmark = pytest.mark.gpu

FULL = ["C3", "C4", "C5", "C5s"]
REF = ["C1", "C2", "C4r", "C5r"]


def _counters(st):
    return [st.total_cell_updates, st.num_regrids, st.hyperbolicity_warnings, st.wet_prefix_repairs]


def _run(z, pb):
    from paper_1803_01450_b200.driver import Simulation
    from paper_1803_01450_b200.errors import CflViolationError
    sim = Simulation(pb)
    rt = lambda: [s.r_t for s in sim.specs]  # noqa: E731

    def cp(prefix):
        st = sim.finish()
        check(z, prefix, gpu_levels(sim), _counters(st), sim.composite_mass(), rt(), st)

    cp("s0_")
    for k in range(1, int(z["done"]) + 1):
        dt = sim.choose_dt()
        assert dt == float(z["dts"][k - 1]), (k, dt, float(z["dts"][k - 1]))
        sim.apply_dynamic_rt(dt)
        sim.advance_coarse_step(dt)
        assert sim.time == float(z[f"s{k}_time"])
        cp(f"s{k}_")
    if "abort_step" in z:
        dt = sim.choose_dt()
        assert dt == float(z["abort_dt"])
        sim.apply_dynamic_rt(dt)
        assert rt() == z["abort_rt"].tolist()
        with pytest.raises(CflViolationError):
            sim.advance_coarse_step(dt)
    sim.close()


@pytest.mark.parametrize("name", FULL)
def test_full_size_matches_oracle(name):
    from make_fullsize import problem
    z = fixture(f"fullsize_{name}.npz")
    if z is None:
        pytest.skip(f"fullsize_{name}.npz not generated")
    _run(z, problem(name))


@pytest.mark.parametrize("name", REF)
def test_config_matches_reference_run(name):
    from make_fullsize import ref_variant
    z = fixture(f"ref_{name}.npz")
    assert z is not None
    _run(z, ref_variant(name)[0])
