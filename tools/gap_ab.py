"""C4 coarse-step device time with and without the bench's instrumentation
(per-launch CUDA events around the finest step and the auxiliary kernels,
the nvidia-smi clock sampler), to size the host-side gaps.

    python tools/gap_ab.py [--steps 10] [--warmup 5] [--modes plain,events,plain]
"""
import argparse
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1803_01450_b200 import problems  # noqa: E402
from paper_1803_01450_b200.driver import Simulation  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=5)
ap.add_argument("--modes", default="plain,events,smi,plain")
a = ap.parse_args()

stream = torch.cuda.Stream()
pb = problems.CONFIGS[a.config]()
sim = Simulation(pb, stream=stream)


def coarse(sim):
    dt = sim.choose_dt()
    sim.apply_dynamic_rt(dt)
    sim.advance_coarse_step(dt)


for _ in range(a.warmup):
    coarse(sim)
for mode in a.modes.split(","):
    smi = None
    if mode == "smi":
        smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "200"],
                               stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    if mode == "events":
        sim.step_timer_level = sim.L
        sim.step_events = []
        sim.kernel_timer = {}
    sim.host_prof.clear()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record(stream)
    for _ in range(a.steps):
        coarse(sim)
    e1.record(stream)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - w0) * 1e3 / a.steps
    ms = e0.elapsed_time(e1) / a.steps
    extra = ""
    if mode == "events":
        st = sum(x.elapsed_time(y) for x, y, _ in sim.step_events) / a.steps
        extra = f" finest-step {st:.2f} ms/step"
        sim.step_timer_level = None
        sim.kernel_timer = None
    if smi is not None:
        smi.terminate()
    host = {k: round(1e3 * v / a.steps, 2) for k, v in sim.host_prof.items()}
    print(f"{mode}: device {ms:.2f} ms/step, wall {wall:.2f} ms/step{extra} host {host}", flush=True)
