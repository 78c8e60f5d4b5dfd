"""Host critical path of a C4 level-3 rebuild: time from the summed-area
table's arrival (the synchronisation in cluster_boxes_device) to the first
kernel of the new pool, split by phase (host perf counters)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1803_01450_b200 import problems, regrid  # noqa: E402
from paper_1803_01450_b200 import driver as D  # noqa: E402
from paper_1803_01450_b200 import device as DV  # noqa: E402

T = {}
marks = []


def wrap(obj, name, label):
    f = getattr(obj, name)

    def w(*a, **k):
        t0 = time.perf_counter()
        r = f(*a, **k)
        marks.append((label, t0, time.perf_counter()))
        return r
    setattr(obj, name, w)


wrap(regrid, "_cluster_from_sat", "bisection")
wrap(D, "chop_boxes", "chop")
wrap(DV.LevelPool, "__init__", "LevelPool()")
wrap(DV.LevelPool, "_build_tiles", "tile list")
wrap(DV.LevelPool, "ghost_plan", "ghost_plan")
wrap(D.Simulation, "_new_pool", "_new_pool (incl. bathy fill/check)")
wrap(D.Simulation, "_rebuild", "_rebuild (total)")
orig_sync = torch.cuda.Stream.synchronize


def tsync(self):
    t0 = time.perf_counter()
    orig_sync(self)
    marks.append(("sync", t0, time.perf_counter()))


torch.cuda.Stream.synchronize = tsync
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
pb = problems.CONFIGS[name]()
sim = D.Simulation(pb, stream=torch.cuda.Stream())
warm, steps = (1, 2) if name == "C5s" else (5, 10)   # C5s meets the CFL guard in its 4th step
for _ in range(warm):
    bench.coarse_step(sim)
marks.clear()
for _ in range(steps):
    bench.coarse_step(sim)
torch.cuda.synchronize()
# per rebuild: phases after the clustering sync
i = 0
while i < len(marks):
    if marks[i][0] == "bisection":
        t_sync_end = max((m[2] for m in marks[:i] if m[0] == "sync"), default=marks[i][1])
        out = {"sync->bisection start": 1e3 * (marks[i][1] - t_sync_end)}
        j = i
        while j < len(marks) and marks[j][0] != "_rebuild (total)":
            out[marks[j][0]] = round(1e3 * (marks[j][2] - marks[j][1]), 3)
            j += 1
        if j < len(marks):
            out["_rebuild end - sync end"] = round(1e3 * (marks[j][2] - t_sync_end), 3)
        print(out)
        i = j
    i += 1
