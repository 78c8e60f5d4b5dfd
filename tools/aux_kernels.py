"""Auxiliary-kernel rooflines (bench.kernel_rooflines) on a config, for A/B
of library variants:  MLAMR_LIB=... python tools/aux_kernels.py [C4] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1803_01450_b200 import problems  # noqa: E402
from paper_1803_01450_b200.driver import Simulation  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
pb = problems.CONFIGS[name]()
st = torch.cuda.Stream()
sim = Simulation(pb, stream=st)
for _ in range(1 if name == "C5s" else 2):   # C5s meets the CFL guard in its 4th step
    bench.coarse_step(sim)
sim.kernel_timer = {}
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(steps):
    bench.coarse_step(sim)
e1.record(st)
torch.cuda.synchronize()
peak = bench._peaks()[0]
tag = os.path.basename(os.environ.get("MLAMR_LIB", "default"))
for k in bench.kernel_rooflines(sim.kernel_timer, peak, e0.elapsed_time(e1) * 1e-3):
    print(f"{tag:12s} {k['kernel']:26s} n={k['launches']:3d} {k['avg_launch_ms']:8.4f} ms  "
          f"{k['achieved_gbs']:7.0f} GB/s  frac {k['frac']:.3f}")
