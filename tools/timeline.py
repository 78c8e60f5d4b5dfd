"""Device timeline of full C4 coarse steps (torch.profiler / CUPTI): kernel
time by kernel, and the GPU-idle gaps between kernels named by the kernels on either side.

    python tools/timeline.py [--config C4] [--steps 10] [--warmup 5] [--out gpurun_out/timeline.json]
"""
import argparse
import collections
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1803_01450_b200 import problems  # noqa: E402
from paper_1803_01450_b200 import driver as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=5)
ap.add_argument("--gap-us", type=float, default=20.0)
ap.add_argument("--out", default="gpurun_out/timeline.json")
a = ap.parse_args()

pb = problems.CONFIGS[a.config]()
stream = torch.cuda.Stream()
sim = D.Simulation(pb, stream=stream)


def coarse(sim):
    dt = sim.choose_dt()
    sim.apply_dynamic_rt(dt)
    sim.advance_coarse_step(dt)


for _ in range(a.warmup):
    coarse(sim)
torch.cuda.synchronize()

t0 = time.perf_counter()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(a.steps):
        coarse(sim)
    torch.cuda.synchronize()
wall = time.perf_counter() - t0

ev = prof.events()
# kineto exposes device activities with time_range on the same clock as the host ranges
kern = sorted([(e.time_range.start, e.time_range.end, e.name) for e in ev if e.device_type.name == "CUDA"])
span = kern[-1][1] - kern[0][0]
busy = 0.0
by = collections.Counter()
cnt = collections.Counter()
gaps = []
end = kern[0][0]
prev = "start"
for s, e, n in kern:
    short = n.split("(")[0].split("<")[0].replace("void ", "")
    if s > end + a.gap_us:
        gaps.append((end, s, prev, short))
    busy += max(0.0, e - max(s, end))
    end = max(end, e)
    prev = short
    by[short] += e - s
    cnt[short] += 1


gap_by = collections.Counter()
for s, e, p0, p1 in gaps:
    gap_by[p0 + " -> " + p1] += e - s
res = {
    "config": a.config, "steps": a.steps, "wall_ms_per_step": 1e3 * wall / a.steps,
    "device_span_ms_per_step": span / 1e3 / a.steps,
    "kernel_busy_ms_per_step": busy / 1e3 / a.steps,
    "idle_ms_per_step": (span - busy) / 1e3 / a.steps,
    "kernels_ms_per_step": {k: round(v / 1e3 / a.steps, 4) for k, v in by.most_common()},
    "launches_per_step": {k: cnt[k] / a.steps for k, _ in by.most_common()},
    "idle_gaps_ms_per_step": {k: round(v / 1e3 / a.steps, 4) for k, v in gap_by.most_common()},
    "n_gaps_per_step": len(gaps) / a.steps,
}
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
with open(a.out, "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res, indent=1))
