import os, sys, time
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import mlamr_oracle as O
from paper_1803_01450_b200 import problems
O.build()
pb = problems.config4()
t0 = time.time(); sim = O.Simulation(pb, workers=os.cpu_count()); t1 = time.time()
print("init", t1 - t0, {l: len(v) for l, v in sim.patches.items()}, "cpus", os.cpu_count(), flush=True)
for k in range(2):
    t1 = time.time(); c0 = sim.stats.total_cell_updates
    dt = sim.choose_dt(); sim.apply_dynamic_rt(dt); sim.advance_coarse_step(dt)
    t2 = time.time(); print("step", k, t2 - t1, "s", (sim.stats.total_cell_updates - c0) * 2 / (t2 - t1), "cell-layer/s", flush=True)
