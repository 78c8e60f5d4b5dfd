"""Where e2e time goes: restore (H2D), K coarse steps, snapshot (D2H)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1803_01450_b200 import problems  # noqa: E402
from paper_1803_01450_b200.driver import Simulation  # noqa: E402

pb = problems.config4()
sim = Simulation(pb)
for _ in range(2):
    sim.advance_coarse_step(sim.choose_dt())
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    snap = sim.snapshot()
    t1 = time.perf_counter()
    sim2 = Simulation.restore(pb, snap)
    Simulation.release_snapshot(snap)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    for _ in range(5):
        sim2.advance_coarse_step(sim2.choose_dt())
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    out = sim2.snapshot()
    t4 = time.perf_counter()
    print(f"rep {rep}: snapshot {1e3*(t1-t0):.1f} ms ({snap['nbytes']/1e9:.2f} GB), restore {1e3*(t2-t1):.1f} ms, "
          f"5 steps {1e3*(t3-t2):.1f} ms, snapshot {1e3*(t4-t3):.1f} ms")
    del sim2, out
