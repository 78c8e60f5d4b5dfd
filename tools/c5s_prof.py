"""Host/device profile of the C5s regrid-stress workload (cProfile of two
coarse steps after one warm-up): where a rebuild of ~76 k patches goes."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1803_01450_b200 import problems  # noqa: E402
from paper_1803_01450_b200.driver import Simulation  # noqa: E402

pb = problems.config5_stress()
sim = Simulation(pb, stream=torch.cuda.Stream())


def coarse():
    dt = sim.choose_dt()
    sim.apply_dynamic_rt(dt)
    sim.advance_coarse_step(dt)


coarse()
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for _ in range(2):
    coarse()
torch.cuda.synchronize()
pr.disable()
print("ms per coarse step", 1e3 * (time.perf_counter() - t0) / 2)
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
