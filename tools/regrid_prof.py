import os, sys, time, collections
sys.path.insert(0, '/root/repo')
import torch
from paper_1803_01450_b200 import problems, regrid, device as DV
from paper_1803_01450_b200 import driver as D
P = collections.defaultdict(float); C = collections.Counter()
orig_sync = torch.cuda.Stream.synchronize
def tsync(self):
    t=time.perf_counter(); orig_sync(self); P['stream.synchronize'] += time.perf_counter()-t; C['stream.synchronize']+=1
torch.cuda.Stream.synchronize = tsync
ocl = regrid._cluster_from_sat
def tcl(*a, **k):
    t=time.perf_counter(); r=ocl(*a, **k); P['bisection'] += time.perf_counter()-t; C['bisection']+=1; return r
regrid._cluster_from_sat = tcl
for name in ['_new_pool','_cluster_level','regrid_from','choose_dt','composite_mass','_sync_status']:
    f = getattr(D.Simulation, name)
    def w(self,*a,f=f,name=name,**k):
        t=time.perf_counter(); r=f(self,*a,**k); P[name]+=time.perf_counter()-t; C[name]+=1; return r
    setattr(D.Simulation, name, w)
og = DV.LevelPool.ghost_plan
def tg(self):
    t=time.perf_counter(); r=og(self); P['ghost_plan'] += time.perf_counter()-t; return r
DV.LevelPool.ghost_plan = tg
pb = problems.config4(); st = torch.cuda.Stream(); sim = D.Simulation(pb, stream=st)
def coarse():
    dt = sim.choose_dt(); sim.apply_dynamic_rt(dt); sim.advance_coarse_step(dt)
for _ in range(5): coarse()
torch.cuda.synchronize(); P.clear(); C.clear()
t=time.perf_counter(); n=10
for _ in range(n): coarse()
torch.cuda.synchronize(); w=time.perf_counter()-t
print('wall ms/step', 1e3*w/n)
for k,v in sorted(P.items(), key=lambda x:-x[1]): print(f'{k:22s} {1e3*v/n:8.2f} ms/step  calls/step {C[k]/n}')

if "--cprofile" in sys.argv:
    import cProfile, pstats
    pr = cProfile.Profile(); pr.enable()
    for _ in range(n): coarse()
    torch.cuda.synchronize(); pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
