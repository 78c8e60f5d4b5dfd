"""Run C5s (problems.config5_stress) for N coarse steps and print r_t, dt
and the regrid count per step (diagnosis helper)."""
import os
import sys
root = sys.argv[1] if len(sys.argv) > 1 else os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
import torch  # noqa: E402
from paper_1803_01450_b200 import problems  # noqa: E402
from paper_1803_01450_b200.driver import Simulation  # noqa: E402
pb = problems.config5()
pb.bernoulli = (0.05,)
pb.flag_rule = ("bernoulli", 0.05, 1)
sim = Simulation(pb)
for k in range(int(sys.argv[2]) if len(sys.argv) > 2 else 12):
    dt = sim.choose_dt()
    sim.apply_dynamic_rt(dt)
    try:
        sim.advance_coarse_step(dt)
    except Exception as e:
        print("step", k, "dt", dt, "rt", [s.r_t for s in sim.specs], "FAILED", e)
        break
    print("step", k, "dt", dt, "rt", [s.r_t for s in sim.specs], "regrids", sim.stats.num_regrids,
          "P2", sim.levels[2].P, flush=True)
