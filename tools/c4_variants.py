"""C4 full schedule under harness variants (cfl / dry tolerance)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1803_01450_b200 import problems  # noqa: E402
from paper_1803_01450_b200.driver import Simulation  # noqa: E402

for spec in sys.argv[1:]:
    kv = dict(x.split("=") for x in spec.split(","))
    pb = problems.config4()
    if "cfl" in kv:
        pb.cfl = float(kv["cfl"])
    if "tol" in kv:
        pb.dry_tolerance = float(kv["tol"])
    n = int(kv.get("n", pb.n_coarse_steps))
    sim = Simulation(pb)
    t0 = time.perf_counter()
    smax = 0.0
    try:
        for k in range(n):
            dt = sim.choose_dt()
            sim.apply_dynamic_rt(dt)
            sim.advance_coarse_step(dt)
            if k % 20 == 19:
                smax = max(smax, float(np.max(sim.level_speed(3))))
        print(spec, "completed", n, "steps to t", round(sim.time, 1), "in", round(time.perf_counter() - t0, 1), "s; max L3 speed seen", round(smax, 1), flush=True)
    except Exception as e:  # noqa: BLE001
        print(spec, "ABORT at step", k, "t", round(sim.time, 1), e, flush=True)
    del sim
