"""Run a config until a CFL abort; report per-step level speeds and, at the
abort, the offending cell's column state (where and why)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1803_01450_b200 import problems  # noqa: E402
from paper_1803_01450_b200.driver import Simulation  # noqa: E402

name = sys.argv[1]
n = int(sys.argv[2])
every = int(sys.argv[3]) if len(sys.argv) > 3 else 5
pb = problems.CONFIGS[name]()
sim = Simulation(pb)
for k in range(n):
    dt = sim.choose_dt()
    sim.apply_dynamic_rt(dt)
    if k % every == 0:
        sp = {lv: round(float(np.max(sim.level_speed(lv))), 1) if sim.levels[lv].P else 0 for lv in sim.levels}
        print(k, "t", round(sim.time, 1), "dt", round(dt, 3), "speeds", sp, flush=True)
    snap = None
    try:
        sim.advance_coarse_step(dt)
    except Exception as e:  # noqa: BLE001
        print("EXC at step", k, e)
        lv = max(sim.levels)
        spl = sim.level_speed(lv)
        i = int(np.argmax(spl))
        box, h, hu, hv, b = sim.patch_fields(lv)[i]
        hi, hui, hvi, bi = h[:, 2:-2, 2:-2], hu[:, 2:-2, 2:-2], hv[:, 2:-2, 2:-2], b[2:-2, 2:-2]
        vel = np.where(hi > pb.dry_tolerance, np.maximum(np.abs(hui), np.abs(hvi)) / np.maximum(hi, 1e-300), 0)
        j = np.unravel_index(np.argmax(vel), vel.shape)
        print("level", lv, "patch", i, "box", box, "max speed", spl[i])
        print("cell", j, "h", hi[:, j[1], j[2]], "hu", hui[:, j[1], j[2]], "hv", hvi[:, j[1], j[2]], "B", bi[j[1], j[2]])
        r0, c0 = max(j[1] - 2, 0), max(j[2] - 2, 0)
        print("h_m around:", np.array2string(hi[j[0], r0:r0 + 5, c0:c0 + 5], precision=4))
        print("B around:", np.array2string(bi[r0:r0 + 5, c0:c0 + 5], precision=2))
        break
