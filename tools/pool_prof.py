"""Host time inside LevelPool construction during C4 coarse steps."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1803_01450_b200 import device as D, problems  # noqa: E402
from paper_1803_01450_b200.driver import Simulation  # noqa: E402

sim = Simulation(problems.config4())
D.POOL_PROF.clear()
t0 = time.perf_counter()
for _ in range(8):
    dt = sim.choose_dt()
    sim.apply_dynamic_rt(dt)
    sim.advance_coarse_step(dt)
torch.cuda.synchronize()
print("wall s", round(time.perf_counter() - t0, 3))
print({k: round(v * 1e3, 1) for k, v in D.POOL_PROF.items()}, D.ALLOC_STATS)
print({k: round(v * 1e3, 1) for k, v in sim.host_prof.items()})
