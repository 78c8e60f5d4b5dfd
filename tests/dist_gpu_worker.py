"""Worker for tests/test_gpu_sharded.py (run under torchrun, gloo backend).

Each rank runs the sharded driver over its share of the patches and, in the
same process, the single-GPU driver over all of them; after every coarse
step every owned patch must be bit-identical, and the all-reduced
statistics must equal the single-GPU ones.  Halfway through, the sharded
run is checkpointed (every rank its own pools) and continued from the
restored copy."""

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def variant(name):
    from paper_1803_01450_b200 import problems
    if name == "C2":
        pb = problems.config2()
        pb.regrid_interval = 2
        return pb, 3
    if name == "C4":
        pb = problems.config4(nx0=64)
        pb.regrid_interval = 2
        return pb, 2
    if name == "C3":
        pb = problems.config3(nx0=32)   # M = 3, gradient flag rule, dynamic r_t
        pb.regrid_interval = 2
        return pb, 3
    if name == "C5":
        pb = problems.config5(nx0=64)
        pb.bernoulli = (0.05,)
        return pb, 3
    raise KeyError(name)


def main():
    name = sys.argv[1]
    from datetime import timedelta
    dist.init_process_group("gloo", timeout=timedelta(seconds=120))
    torch.cuda.set_device(0)
    from paper_1803_01450_b200.driver import Simulation
    from paper_1803_01450_b200.sharded import ShardedSimulation
    pb, steps = variant(name)
    ref = Simulation(pb, stream=torch.cuda.Stream())
    sh = ShardedSimulation(pb, stream=torch.cuda.Stream())
    rank = dist.get_rank()

    def compare(tag):
        bad = 0
        for lev in range(1, ref.L + 1):
            if lev not in ref.levels:
                continue
            full = ref.patch_fields(lev)
            gl = sh.layout.get(lev, np.zeros((0, 4)))
            assert [tuple(int(v) for v in b) for b in gl] == [f[0] for f in full], (tag, lev, "layout")
            for g, (box, h, hu, hv, b) in sh.owned_fields(lev).items():
                R = full[g]
                for a, c in ((h, R[1]), (hu, R[2]), (hv, R[3])):
                    x, y = a[:, 2:-2, 2:-2], c[:, 2:-2, 2:-2]
                    if not np.array_equal(x, y):
                        bad += 1
                        if os.environ.get("MLAMR_TEST_VERBOSE"):
                            d = np.argwhere(x != y)
                            print(f"rank {rank} {tag}: level {lev} patch {g} box {box} differs in {len(d)} cells, "
                                  f"first {d[:4].tolist()}, max |diff| {np.nanmax(np.abs(x - y)):.3e}\n"
                                  + "\n".join("".join(".X"[int(v)] for v in row) for row in (x != y).any(axis=0)),
                                  flush=True)
        assert bad == 0, (tag, rank, bad)

    compare("init")
    for k in range(steps):
        if k == steps // 2:
            # checkpoint: every rank snapshots its own pools (owned +
            # shadows); the restored sharded run continues bit-identically
            snap = sh.snapshot()
            sh.close()
            sh = ShardedSimulation.restore(pb, snap, stream=torch.cuda.Stream())
            compare(f"restored before step{k}")
        dt = ref.choose_dt()
        assert sh.choose_dt() == dt, k
        ref.apply_dynamic_rt(dt)
        sh.apply_dynamic_rt(dt)
        ref.advance_coarse_step(dt)
        sh.advance_coarse_step(dt)
        compare(f"step{k}")
    # frames: rank 0 assembles every rank's owned records into the bytes
    # the single-GPU driver writes
    from paper_1803_01450_b200 import frames as F
    fb = F.frame_bytes(sh)
    fa = F.frame_bytes(ref)
    if rank == 0:
        assert fb == fa, ("frame", len(fa), len(fb or b""))
    else:
        assert fb is None
    a, b = ref.finish(), sh.finish()
    assert a.total_cell_updates == b.total_cell_updates, (a.total_cell_updates, b.total_cell_updates)
    assert a.cell_updates_per_level == b.cell_updates_per_level, (a.cell_updates_per_level,
                                                                  b.cell_updates_per_level)
    assert a.num_regrids == b.num_regrids
    # sync_delta = mass - mass_prev - (refine + derefine delta) per coarse step
    # (driver.py:303-307): the sharded event delta is all-reduced like the mass
    scale = float(np.abs(ref.composite_mass()).sum())
    np.testing.assert_allclose(b.sync_delta, a.sync_delta, rtol=0, atol=1e-11 * scale)
    for x, y in ((a.refine_delta, b.refine_delta), (a.derefine_delta, b.derefine_delta),
                 (a.clipped_mass, b.clipped_mass)):
        np.testing.assert_allclose(np.asarray(y, float), np.asarray(x, float), rtol=0, atol=1e-11 * scale)
    # finish() is idempotent: a second call returns the same global numbers
    c = sh.finish()
    assert c.total_cell_updates == b.total_cell_updates and c.cell_updates_per_level == b.cell_updates_per_level
    assert c.refine_delta == b.refine_delta and c.clipped_mass == b.clipped_mass
    np.testing.assert_allclose(sh.composite_mass(), ref.composite_mass(), rtol=1e-12)
    if sh.overlap_refresh:
        # the finest level ran its refresh (i) overlapped: some tiles before
        # the exchange completed, the rest after it
        fp = sh.levels[sh.L]
        assert 0 < fp._n_indep < fp.n_tiles, (fp._n_indep, fp.n_tiles)
        print(f"rank {rank}: finest tiles stepped during the exchange {fp._n_indep} of {fp.n_tiles}", flush=True)
    print(f"rank {rank}: {name} sharded == single-GPU ({steps} steps, exchanged {sh.bytes_exchanged} B, "
          f"owned {[int(p.n_owned) for p in sh.levels.values()]} of {[len(v) for v in sh.layout.values()]})",
          flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
