"""Is the step kernel (K1) bound by HBM or by its arithmetic?

Times the finest-level step launch of C4 with CUDA events over three tile
lists of the same length: the real one (3.7 GB of compulsory HBM traffic
per launch); `--hot` distinct tiles spread evenly over the level, repeated
(the same mix of all-wet / general-path / patch-edge tiles as the real
list, but a working set that stays in L2, so almost no HBM traffic); and
`--hot` adjacent tiles repeated (a few patches only -- their tile mix is
not representative, e.g. all-wet deep water, so this one is a lower bound,
not a fair comparison).  Both launches take the fused-sibling path the
driver uses.  Round 1, B200: real 3.19 ms, spread-64 2.99 ms (94 %),
spread-256 95 %, spread-1024 100 %, adjacent-64 2.24 ms (70 %): the launch
is not limited by HBM bandwidth or latency.

    python tools/compute_bound.py [--nx0 512] [--reps 5] [--hot 64]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1803_01450_b200 import problems  # noqa: E402
from paper_1803_01450_b200.driver import Simulation  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nx0", type=int, default=512)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--hot", type=int, default=64, help="distinct tiles in the L2-resident list")
a = ap.parse_args()

sim = Simulation(problems.config4(nx0=a.nx0))
sim.advance_coarse_step(sim.choose_dt())
L = sim.L
pool = sim.levels[L]
gbase, plan = pool.ghost_plan()[:2]
src, dst = pool.state, pool.other
lv = pool.struct(src)
dt = 1e-3
n = pool.n_tiles
hot = pool.tiles_d.view(-1, 3)[:a.hot].repeat((n + a.hot - 1) // a.hot, 1)[:n].contiguous()


def run(tiles):
    ev = []
    for r in range(a.reps + 1):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(sim.stream)
        sim._call(sim.lib.mlamr_step, lv, src.data_ptr(), dst.data_ptr(), tiles.data_ptr(), n, pool.tile_tx, dt, 0,
                  sim.prm, pool.speed_bits.data_ptr(), pool.tile_acc.data_ptr(), sim.status.data_ptr(),
                  gbase.data_ptr(), plan.data_ptr(), sim.sh)
        e1.record(sim.stream)
        ev.append((e0, e1))
    torch.cuda.synchronize()
    return float(np.mean([x.elapsed_time(y) for x, y in ev[1:]]))


# the same number of distinct tiles, spread evenly over the whole level
# (L2-resident data, but every tile in other pages: separates the cost of
# DRAM latency/bandwidth from address-translation misses)
all_t = pool.tiles_d.view(-1, 3)
spread = all_t[torch.linspace(0, n - 1, a.hot, device=all_t.device).long()]
spread = spread.repeat((n + a.hot - 1) // a.hot, 1)[:n].contiguous()

t_real = run(pool.tiles_d)
t_hot = run(hot)
t_spread = run(spread)
t_real2 = run(pool.tiles_d)
print(f"tiles {n}: real tile list {t_real:.3f} / {t_real2:.3f} ms, L2-resident list ({a.hot} adjacent tiles) "
      f"{t_hot:.3f} ms ({100 * t_hot / t_real:.0f}%), {a.hot} tiles spread over the level {t_spread:.3f} ms "
      f"({100 * t_spread / t_real:.0f}%)")
