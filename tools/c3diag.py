"""C3 robustness probe: per coarse step dt, r_t, level speeds; on a CFL
abort, the offending patch's largest velocity and its column state."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1803_01450_b200 import problems  # noqa: E402
from paper_1803_01450_b200.driver import Simulation  # noqa: E402

nx0 = int(sys.argv[1]) if len(sys.argv) > 1 else 256
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
pb = problems.config3(nx0=nx0)
sim = Simulation(pb)
for k in range(nsteps):
    dt = sim.choose_dt()
    sim.apply_dynamic_rt(dt)
    sp = {lv: float(np.max(sim.level_speed(lv))) if sim.levels[lv].P else 0 for lv in sim.levels}
    print(k, "t", round(sim.time, 2), "dt", round(dt, 3), "rt", [s.r_t for s in sim.specs],
          "speeds", {lv: round(v, 1) for lv, v in sp.items()}, "P", {lv: p.P for lv, p in sim.levels.items()},
          flush=True)
    try:
        sim.advance_coarse_step(dt)
    except Exception as e:  # noqa: BLE001
        print("EXC", e)
        for lv in sorted(sim.levels, reverse=True):
            spl = sim.level_speed(lv)
            i = int(np.argmax(spl))
            print("level", lv, "max speed", spl[i], "patch", i, sim.levels[lv].boxes[i])
        break
