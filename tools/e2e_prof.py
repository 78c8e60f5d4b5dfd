"""Where e2e time goes: restore (H2D), K coarse steps, snapshot (D2H).

    python tools/e2e_prof.py [--keep]   (--keep: the source simulation stays
                                         alive, holding its device memory)
"""
import cProfile
import gc
import os
import pstats
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
snap0 = sim.snapshot()
if "--keep" not in sys.argv:
    del sim
    gc.collect()
for rep in range(2):
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    prof = cProfile.Profile() if rep == 1 else None
    if prof:
        prof.enable()
    sim2 = Simulation.restore(pb, snap0)
    torch.cuda.synchronize()
    if prof:
        prof.disable()
    t2 = time.perf_counter()
    for _ in range(5):
        sim2.advance_coarse_step(sim2.choose_dt())
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    out = sim2.snapshot()
    t4 = time.perf_counter()
    print(f"rep {rep}: restore {1e3*(t2-t1):.1f} ms ({snap0['nbytes']/1e9:.2f} GB), "
          f"5 steps {1e3*(t3-t2):.1f} ms, snapshot {1e3*(t4-t3):.1f} ms")
    if prof:
        pstats.Stats(prof).sort_stats("cumtime").print_stats(18)
    Simulation.release_snapshot(out)
    del sim2, out
    gc.collect()
