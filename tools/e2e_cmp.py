"""Original vs restored simulation: per-step device (events) and wall time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
clk = bench.ClockSampler(0)
import torch
from paper_1803_01450_b200 import problems, device as D
from paper_1803_01450_b200.driver import Simulation
pb = problems.config4()
stream = torch.cuda.Stream()
def run(sim, n, tag):
    sim.host_prof.clear()
    a0 = dict(D.ALLOC_STATS)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    clk.__enter__()
    e0.record(sim.stream)
    for _ in range(n):
        dt = sim.choose_dt(); sim.apply_dynamic_rt(dt); sim.advance_coarse_step(dt)
    e1.record(sim.stream)
    torch.cuda.synchronize()
    clk.__exit__()
    w = 1e3 * (time.perf_counter() - t0) / n
    print(f"{tag}: events {e0.elapsed_time(e1) / n:.1f} ms/step, wall {w:.1f} ms/step, cells {sim.stats.total_cell_updates}",
          "alloc", {k: v - a0.get(k, 0) for k, v in D.ALLOC_STATS.items()})
    print("   ", clk.summary())
    print("   ", {k: round(1e3 * v / n, 1) for k, v in sim.host_prof.items()})
sim = Simulation(pb, stream=stream)
run(sim, 3, "warm")
run(sim, 5, "orig")
snap = sim.snapshot()
sim.close()
del sim
import gc
gc.collect()
torch.cuda.synchronize()
t0 = time.perf_counter()
a0 = dict(D.ALLOC_STATS)
sim2 = Simulation.restore(pb, snap, stream=stream)
Simulation.release_snapshot(snap)
torch.cuda.synchronize()
print(f"restore {1e3 * (time.perf_counter() - t0):.1f} ms", {k: v - a0.get(k, 0) for k, v in D.ALLOC_STATS.items()})
for i in range(5):
    run(sim2, 1, f"restored step {i}")
t0 = time.perf_counter()
out = sim2.snapshot()
print(f"snapshot {1e3 * (time.perf_counter() - t0):.1f} ms")
clk.stop()
