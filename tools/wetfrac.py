import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_1803_01450_b200 import problems
from paper_1803_01450_b200.driver import Simulation
pb = problems.config4()
sim = Simulation(pb)
for _ in range(3):
    sim.advance_coarse_step(sim.choose_dt())
tol = pb.dry_tolerance
for lev in (2, 3):
    tot = wet = 0
    for box, h, hu, hv, b in sim.patch_fields(lev):
        ny, nx = h.shape[1] - 4, h.shape[2] - 4
        for j0 in range(0, ny, 16):
            for i0 in range(0, nx, 32):
                sub = h[:, 1 + j0:min(j0 + 16, ny) + 3, 1 + i0:min(i0 + 32, nx) + 3]
                tot += 1
                wet += bool((sub > tol).all())
    print("level", lev, "tiles", tot, "all-wet fraction", wet / tot)
