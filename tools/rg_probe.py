import sys; sys.path.insert(0,'/root/repo')
import numpy as np, torch
from paper_1803_01450_b200 import problems, driver as D
orig = D.regrid_fill_bytes
def spy(nb, ob, rx, ry, M):
    nb=np.asarray(nb); tot=int(((nb[:,2]-nb[:,0]+1)*(nb[:,3]-nb[:,1]+1)).sum())
    b=orig(nb, ob, rx, ry, M)
    # solve for copied: b = 8*(3M+1+(3M+1)/(rx ry))*(tot-c) + 96*c
    a=8*(3*M+1+(3*M+1)/(rx*ry)); c=(b - a*tot)/(8*6*M - a)
    print(f"rebuild: new cells {tot}, copied {c:.0f} ({c/tot:.1%}), refined {tot-c:.0f}")
    return b
D.regrid_fill_bytes = spy
import bench
pb = problems.config4(); st = torch.cuda.Stream(); sim = D.Simulation(pb, stream=st)
sim.kernel_timer = {}
for _ in range(12): bench.coarse_step(sim)
torch.cuda.synchronize()
for name, evs in sim.kernel_timer.items():
    if 'regrid' in name:
        for a,b_,n in evs: print(name, round(a.elapsed_time(b_),3), "ms", (n() if callable(n) else n)/1e9, "GB")
