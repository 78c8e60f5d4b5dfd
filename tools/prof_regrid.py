"""cProfile of host-side regrid work on C4 (which Python calls dominate)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1803_01450_b200 import problems  # noqa: E402
from paper_1803_01450_b200.driver import Simulation  # noqa: E402

nx0 = int(sys.argv[1]) if len(sys.argv) > 1 else 512
sim = Simulation(problems.config4(nx0=nx0))
sim.advance_coarse_step(sim.choose_dt())
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    sim._rebuild(2)
    torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
print(dict(sim.host_prof))
