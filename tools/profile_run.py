"""Small driver for ncu: a few coarse steps of a (down-scaled) config.

    python tools/profile_run.py [--config C4] [--nx0 128] [--steps 1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1803_01450_b200 import problems  # noqa: E402
from paper_1803_01450_b200.driver import Simulation  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--nx0", type=int, default=128)
ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()
if a.config == "C4":
    pb = problems.config4(nx0=a.nx0)
else:
    pb = problems.CONFIGS[a.config]()
sim = Simulation(pb)
for _ in range(a.steps):
    dt = sim.choose_dt()
    sim.apply_dynamic_rt(dt)
    sim.advance_coarse_step(dt)
torch.cuda.synchronize()
print("ok", {k: v.P for k, v in sim.levels.items()}, sim.stats.total_cell_updates)
