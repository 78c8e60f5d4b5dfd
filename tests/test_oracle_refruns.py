"""The oracle against the REFERENCE's own runs of the BASELINE
configurations (tests/golden/make_refruns.py: C1 and C2 at full size, C2
over its whole 50-step schedule with regrids every 5; C4 and C5 reduced to
L1 64x64 with regrids; C5's run ends in the reference's own CFL abort).
Layouts and every patch interior bit-exact, dt and counters equal, mass
diagnostics to 1e-11 of the mass scale."""

import numpy as np
import pytest

from fixture_runs import check, fixture, oracle_levels


def _stats(sim):
    st = sim.stats
    return [st.total_cell_updates, st.num_regrids, st.hyperbolicity_warnings, st.wet_prefix_repairs]


@pytest.mark.parametrize("name", ["C1", "C2", "C4r", "C5r"])
def test_oracle_matches_reference_run(oracle, name):
    from make_fullsize import ref_variant
    z = fixture(f"ref_{name}.npz")
    assert z is not None, f"ref_{name}.npz missing"
    pb, _ = ref_variant(name)
    sim = oracle.Simulation(pb)
    rt = lambda: [s.r_t for s in sim.specs]  # noqa: E731
    check(z, "s0_", oracle_levels(sim), _stats(sim), sim.composite_mass(), rt(), sim.stats)
    for k in range(1, int(z["done"]) + 1):
        dt = sim.choose_dt()
        assert dt == float(z["dts"][k - 1]), (k, dt)
        sim.apply_dynamic_rt(dt)
        sim.advance_coarse_step(dt)
        assert sim.time == float(z[f"s{k}_time"])
        check(z, f"s{k}_", oracle_levels(sim), _stats(sim), sim.composite_mass(), rt(), sim.stats)
    if "abort_step" in z:
        dt = sim.choose_dt()
        assert dt == float(z["abort_dt"])
        sim.apply_dynamic_rt(dt)
        assert rt() == z["abort_rt"].tolist()
        with pytest.raises(oracle.CflViolation) as ei:
            sim.advance_coarse_step(dt)
        # the same patch and Courant number as the reference's message
        msg = str(z["abort_msg"])
        assert msg.split(" on level")[0] == str(ei.value).split(" on level")[0]
        box = msg.split("IndexBox(")[1].rstrip(")")
        want = tuple(int(kv.split("=")[1]) for kv in box.split(", "))
        assert f"Box(lo_i={want[0]}, lo_j={want[1]}, hi_i={want[2]}, hi_j={want[3]})" in str(ei.value)
