"""Every BASELINE configuration at full size for its full schedule of
coarse steps on one GPU: wall time, updates, regrids and the mass
identity residual (a robustness check, not the bench)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1803_01450_b200 import problems  # noqa: E402
from paper_1803_01450_b200.driver import Simulation  # noqa: E402

names = sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]
for name in names:
    pb = problems.CONFIGS[name]()
    t0 = time.perf_counter()
    sim = Simulation(pb)
    t1 = time.perf_counter()
    st = sim.run(pb.n_coarse_steps)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    res = [st.final_mass[m] - st.initial_mass[m] - (st.refine_delta[m] + st.derefine_delta[m] + st.sync_delta[m])
           for m in range(pb.num_layers)]
    rel = max(abs(r) / max(abs(st.initial_mass[m]), 1e-300) for m, r in enumerate(res))
    print(f"{name}: {st.num_coarse_steps} coarse steps to t={sim.time:.6g} in {t2 - t1:.2f} s (setup {t1 - t0:.1f} s), "
          f"{st.total_cell_updates * pb.num_layers:.4g} cell-layer updates "
          f"({st.total_cell_updates * pb.num_layers / (t2 - t1):.3g}/s), regrids {st.num_regrids}, "
          f"patches {[p.P for p in sim.levels.values()]}, mass-identity residual {rel:.2e} (relative)", flush=True)
    del sim
