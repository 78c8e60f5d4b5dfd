import sys; sys.path.insert(0,'/root/repo')
import numpy as np, torch
from paper_1803_01450_b200 import problems
from paper_1803_01450_b200.driver import Simulation
pb = problems.config4(); st = torch.cuda.Stream(); sim = Simulation(pb, stream=st)
for _ in range(3):
    dt = sim.choose_dt(); sim.advance_coarse_step(dt)
for lev in (1,2,3):
    sim.step_timer_level = lev; sim.step_events = []
    for _ in range(2):
        dt = sim.choose_dt(); sim.advance_coarse_step(dt)
    torch.cuda.synchronize()
    d = [a.elapsed_time(b) for a,b,_ in sim.step_events]
    p = sim.levels[lev]
    print("level", lev, "P", p.P, "cells", p.ncells, "tiles", p.n_tiles, "tile_tx", p.tile_tx, "launches", len(d), "avg ms %.3f" % np.mean(d), "Gcell/s %.2f" % (p.ncells/np.mean(d)/1e6))
