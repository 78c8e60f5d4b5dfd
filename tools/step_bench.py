"""Average finest-level step-kernel time (CUDA events) on a down-scaled C4.

    MLAMR_LIB=path/to/variant.so python tools/step_bench.py [--nx0 256] [--steps 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1803_01450_b200 import problems  # noqa: E402
from paper_1803_01450_b200.driver import Simulation  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nx0", type=int, default=256)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
pb = problems.config4(nx0=a.nx0)
sim = Simulation(pb)
sim.advance_coarse_step(sim.choose_dt())
sim.step_timer_level = sim.L
sim.step_events = []
for _ in range(a.steps):
    sim.advance_coarse_step(sim.choose_dt())
torch.cuda.synchronize()
d = [e0.elapsed_time(e1) for e0, e1, _ in sim.step_events]
P = sim.levels[sim.L]
b = P.boxes
nx = b[:, 2] - b[:, 0] + 1
ny = b[:, 3] - b[:, 1] + 1
byts = int((8 * (7 * (nx + 2) * (ny + 2) + 6 * nx * ny)).sum())
print(f"{os.environ.get('MLAMR_LIB') or 'default'}: L3 patches {P.P} tiles {P.n_tiles} "
      f"step {np.mean(d):.3f} ms (min {np.min(d):.3f}) -> {byts / np.mean(d) / 1e6:.0f} GB/s")
