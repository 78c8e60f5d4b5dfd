#!/usr/bin/env python
"""Benchmark: multilayer AMR cell-layer updates/s (regrid + ghost fill +
patch step + coarsen) on the BASELINE configuration C4, plus the step
kernel's fraction of the B200 HBM roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config C4] [--no-e2e] [--no-cpu-baseline]

A "step" is one coarse AMR step: level-1 dt reduction, regrid when due,
the subcycled ghost fills / patch steps of all levels and the coarsenings
(driver.py:299-309 of the reference).  The reference arm (``--impl
reference``) times the oracle port of the reference's CPU algorithm
(oracle/, C + numpy, all host threads) on a bounded sample of the same
workload.  Multi-GPU (torchrun, N>1): one C4 problem whose patches are sharded along a Morton curve (sharded.py),
shadow halos move over NCCL, and the timed region is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "multilayer AMR cell-layer updates/s (regrid + patch step), % of HBM roofline"
UNIT = "cell-layer updates/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms by ONE
    long-running nvidia-smi process (started before CUDA is initialised, so
    no fork of a large process happens inside the timed region); a reader
    thread timestamps the lines and :meth:`window` selects those inside the
    timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.lines = []
        self.proc = None
        self.t0 = self.t1 = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), [x.strip() for x in line.split(",")]))

    def __enter__(self):
        self.t0 = time.time()
        return self

    def __exit__(self, *a):
        self.t1 = time.time() + 0.25

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()

    def summary(self):
        samples = [v for (t, v) in self.lines if self.t0 is not None and self.t0 <= t <= (self.t1 or t)]
        if not samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        num = lambda x: x.replace(".", "").isdigit()
        sm = sorted(float(s[0]) for s in samples if num(s[0]))
        mx = max((float(s[1]) for s in samples if num(s[1])), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in samples for k in range(4)
                          if len(s) > 3 + k and s[3 + k].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(samples)}


def coarse_step(sim):
    dt = sim.choose_dt()
    sim.apply_dynamic_rt(dt)
    sim.advance_coarse_step(dt)


def kernel_rooflines(timer, peak, span_s):
    """Per-kernel roofline of the auxiliary kernels timed in the region:
    algorithmic bytes (driver.py's _kt1 call sites) over
    the CUDA-event launch durations, against the HBM peak."""
    out = []
    for name, evs in sorted((timer or {}).items()):
        durs = [a.elapsed_time(b) * 1e-3 for a, b, _ in evs]
        byts = [int(n() if callable(n) else n) for _, _, n in evs]
        if not durs or sum(durs) <= 0:
            continue
        gbs = sum(byts) / sum(durs) / 1e9
        out.append({"kernel": name, "launches": len(durs), "avg_launch_ms": 1e3 * sum(durs) / len(durs),
                    "bytes_per_launch": int(sum(byts) / len(byts)), "achieved_gbs": gbs,
                    "frac": gbs / peak, "share_of_step": sum(durs) / span_s})
    return out


def stress_run(stream, steps: int, warmup: int, peak):
    """C5s (problems.config5_stress): C5 with Bernoulli(0.05) flags, so the
    level-2 layout is rebuilt -- refine, copy, derefine -- every coarse step.
    Device-timed like the main line; reported inside it."""
    import torch
    from paper_1803_01450_b200 import problems
    from paper_1803_01450_b200.driver import Simulation
    pb = problems.config5_stress()
    sim = Simulation(pb, stream=stream)
    for _ in range(warmup):
        coarse_step(sim)
    sim.kernel_timer = {}
    sim.step_timer_level = sim.L
    sim.step_events = []
    r0, c0 = sim.stats.num_regrids, sim.stats.total_cell_updates
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        coarse_step(sim)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    cells = (sim.stats.total_cell_updates - c0) * pb.num_layers
    durs = [a.elapsed_time(b) * 1e-3 for a, b, _ in sim.step_events]
    byts = [step_bytes(p, pb.num_layers) for _, _, p in sim.step_events]
    res = {"workload": "C5s: C5 (L1 1280^2, r=(4,2), 16x16 patches, dynamic r_t) with Bernoulli(0.05) flags",
           "value": cells / (ms * 1e-3), "unit": UNIT, "steps": steps, "warmup": warmup,
           "ms_per_step": ms / steps, "regrids_per_step": (sim.stats.num_regrids - r0) / steps,
           "patches_level2": int(sim.levels[2].P) if 2 in sim.levels else 0,
           "step_kernel": {"avg_launch_ms": 1e3 * float(sum(durs) / len(durs)) if durs else None,
                           "achieved_gbs": sum(byts) / sum(durs) / 1e9 if durs else None,
                           "share_of_step": sum(durs) / (ms * 1e-3) if durs else None},
           "kernels": kernel_rooflines(sim.kernel_timer, peak, ms * 1e-3)}
    sim.close()
    return res


def step_bytes(pool, M):
    """Algorithmic HBM bytes of one step launch on a level:
    8*[(3M+1)*(nx+2)(ny+2) + 3M*nx*ny] per stepped (owned) patch."""
    b = pool.boxes if pool.owned is None else pool.boxes[pool.owned]
    nx = b[:, 2] - b[:, 0] + 1
    ny = b[:, 3] - b[:, 1] + 1
    return int((8 * ((3 * M + 1) * (nx + 2) * (ny + 2) + 3 * M * nx * ny)).sum())


# ---------------------------------------------------------------------------
# reference arm: the oracle port of the reference's CPU algorithm
# ---------------------------------------------------------------------------
def cpu_sample_problem(name: str, scale_nx0: int):
    from paper_1803_01450_b200 import problems
    if name == "C4":
        return problems.config4(nx0=scale_nx0), f"C4 generator at L1 {scale_nx0}x{scale_nx0} " \
                                                f"(dx as C4, {scale_nx0 ** 2 / 512 ** 2:.4f} of C4's area)"
    return problems.CONFIGS[name](), name


def run_cpu(name: str, steps: int, warmup: int, workers: int, scale_nx0: int):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import mlamr_oracle
    mlamr_oracle.build()
    pb, desc = cpu_sample_problem(name, scale_nx0)
    sim = mlamr_oracle.Simulation(pb, workers=workers)
    for _ in range(warmup):
        coarse_step(sim)
    c0 = sim.stats.total_cell_updates
    t0 = time.perf_counter()
    for _ in range(steps):
        coarse_step(sim)
    t = time.perf_counter() - t0
    cells = (sim.stats.total_cell_updates - c0) * pb.num_layers
    return cells / t, t, desc, sim


def reference_arm(args):
    """The reference's CPU algorithm (the oracle port: C + numpy, one worker
    thread per host core, as the reference's ThreadPool) on the SAME
    workload as the GPU arm -- the full configuration, not a down-scaled
    one.  The oracle keeps the reference's per-patch Python orchestration,
    so a full C4 coarse step takes ~110 s on 16 cores: the arm times whole
    coarse steps from the initial hierarchy until a time budget is used, at
    least one, and reports the rate of those."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import mlamr_oracle
    from paper_1803_01450_b200 import problems
    mlamr_oracle.build()
    workers = os.cpu_count() or 1
    budget = float(os.environ.get("MLAMR_REF_BUDGET_S", "150"))
    pb = problems.CONFIGS[args.config]()
    t_init = time.perf_counter()
    sim = mlamr_oracle.Simulation(pb, workers=workers)
    t_init = time.perf_counter() - t_init
    # no warm-up steps: the CPU code has nothing to warm beyond the untimed
    # initialisation (library loaded, hierarchy built), and one full C4
    # step is ~2 minutes of the budget
    warm = 0
    c0 = sim.stats.total_cell_updates
    t0 = time.perf_counter()
    steps = 0
    last = 0.0
    # another step only if it is expected to end inside the budget
    while steps < max(1, args.steps) and (steps == 0 or time.perf_counter() - t0 + last < budget):
        ts = time.perf_counter()
        coarse_step(sim)
        last = time.perf_counter() - ts
        steps += 1
    t = time.perf_counter() - t0
    v = (sim.stats.total_cell_updates - c0) * pb.num_layers / t
    desc = (f"{args.config} full size ({ {l: len(ps) for l, ps in sim.patches.items()} } patches per level); "
            f"{steps} timed coarse steps after {warm} warm-up (of {args.steps} + {args.warmup} requested: "
            f"time budget {budget:.0f} s); init {t_init:.1f} s untimed; oracle/ C+numpy port, {workers} threads")
    workload = (f"{args.config}: {pb.num_levels} levels, M={pb.num_layers}, L1 {pb.coarse_nx}x{pb.coarse_ny}, "
                f"ratios {pb.ratios_x}")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload, "sample": desc},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": workers, "kind": "port", "sample": desc},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def b200_arm(args):
    local0 = int(os.environ.get("LOCAL_RANK", "0"))
    clk = ClockSampler(local0)   # before CUDA initialisation
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1803_01450_b200 import _native as N
    from paper_1803_01450_b200 import problems
    from paper_1803_01450_b200.driver import Simulation

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("MLAMR_DIST_BACKEND", "nccl")   # gloo: test ranks sharing one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    pb = problems.CONFIGS[args.config]()
    M = pb.num_layers
    stream = torch.cuda.Stream()
    if world > 1:
        # SFC-sharded patches over NCCL (strong scaling: one C4 problem)
        from paper_1803_01450_b200.sharded import ShardedSimulation
        dist.barrier()
        sim = ShardedSimulation(pb, stream=stream)
    else:
        sim = Simulation(pb, stream=stream)
    L = sim.L
    for _ in range(args.warmup):
        coarse_step(sim)

    # ---- timed region: K coarse steps, device clock ----------------------
    sim.host_prof.clear()
    from paper_1803_01450_b200 import device as _D
    _D.POOL_PROF.clear()
    # only the finest step launches carry events inside the timed region (16
    # pairs per coarse step); the auxiliary kernels' per-launch events and
    # byte accounting cost ~4 ms per C4 coarse step (tools/gap_ab.py) and run
    # in a pass of their own after it
    sim.step_timer_level = L
    sim.step_events = []
    sim.kernel_timer = None
    launches0 = N.LAUNCHES[0]
    cells0 = sim.stats.total_cell_updates
    xbytes0 = getattr(sim, "bytes_exchanged", 0)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    prof = None
    if os.environ.get("MLAMR_CPROFILE"):
        import cProfile
        prof = cProfile.Profile()
        prof.enable()
    with clk:
        e0.record(stream)
        for _ in range(args.steps):
            coarse_step(sim)
        e1.record(stream)
        torch.cuda.synchronize()
    if prof is not None:
        import pstats
        prof.disable()
        pstats.Stats(prof, stream=sys.stderr).sort_stats("tottime").print_stats(20)
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    cells = (sim.stats.total_cell_updates - cells0) * M
    launches = N.LAUNCHES[0] - launches0
    t_max = ms
    cells_all = cells
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
        cc = torch.tensor([cells], dtype=torch.float64, device="cuda")
        dist.all_reduce(cc, op=dist.ReduceOp.SUM)
        cells_all = float(cc.item())
    value = cells_all / (t_max * 1e-3)
    if os.environ.get("MLAMR_POOL_PROF"):
        print("pool_prof_ms", {k: round(1e3 * v, 2) for k, v in _D.POOL_PROF.items()}, file=sys.stderr)

    # ---- roofline of the dominant kernel (finest-level step) --------------
    durs, byts = [], []
    for a, b, pool in sim.step_events:
        durs.append(a.elapsed_time(b) * 1e-3)
        byts.append(step_bytes(pool, M))
    peak, peak_kind = _peaks()
    traffic, traffic_ratio = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "step_traffic.json")) as f:
            tj = json.load(f)
        traffic, traffic_ratio = tj["dram_bytes"], tj["traffic_over_algorithmic"]
    except Exception:
        pass
    achieved = (sum(byts) / sum(durs)) / 1e9 if durs else None
    step_share = sum(durs) / (ms * 1e-3) if durs else None
    sim.step_timer_level = None
    pool_bytes = sum(p.state.numel() * 8 * 2 + p.bathy.numel() * 8 for p in sim.levels.values())
    patches_per_level = ({str(k): int(len(v)) for k, v in sim.layout.items()}
                         if world > 1 else {str(k): v.P for k, v in sim.levels.items()})
    cells_per_level = {str(k): v.ncells for k, v in sim.levels.items()}
    host_ms = {k: round(1e3 * v / args.steps, 2) for k, v in sim.host_prof.items()}
    xbytes = int((getattr(sim, "bytes_exchanged", 0) - xbytes0) / args.steps)
    # ---- auxiliary kernels: an instrumented pass outside the timed region ----
    kernels = None
    if not args.no_aux:
        sim.kernel_timer = {}
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        n_aux = max(1, min(args.steps, 10))
        for _ in range(n_aux):
            coarse_step(sim)
        a1.record(stream)
        torch.cuda.synchronize()
        kernels = kernel_rooflines(sim.kernel_timer, peak, a0.elapsed_time(a1) * 1e-3)
        sim.kernel_timer = None

    # ---- regrid stress (C5s), single GPU --------------------------------------
    stress = None
    if world == 1 and not args.no_stress and args.config == "C4":
        # C5s's dynamic-r_t harness rule meets the CFL guard in its 4th coarse
        # step (t = 19.17; the pre-change tree does the same): warm-up 1 + 2
        # timed steps, each with a level-2 rebuild
        stress = stress_run(stream, 2, 1, peak)

    # ---- e2e: host buffers -> device -> K steps -> host ---------------------
    e2e = None
    if not args.no_e2e:
        snap = sim.snapshot()
        # the user's checkpoint/restore cycle in one process: the source
        # simulation hands its device buffers back for the restored one
        # (under sharding every rank snapshots and restores its own pools)
        sim.close()
        del sim
        import gc
        gc.collect()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        if world > 1:
            sim2 = ShardedSimulation.restore(pb, snap, stream=stream)
        else:
            sim2 = Simulation.restore(pb, snap, stream=stream)
        Simulation.release_snapshot(snap)   # its pinned buffers take the final snapshot
        c0 = sim2.stats.total_cell_updates
        for _ in range(args.steps):
            coarse_step(sim2)
        out = sim2.snapshot()
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        ce = (sim2.stats.total_cell_updates - c0) * M
        hb, db = sim2.h2d_bytes, sim2.d2h_bytes
        if world > 1:
            tt = torch.tensor([te], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
            cc = torch.tensor([ce, hb, db], dtype=torch.float64, device="cuda")
            dist.all_reduce(cc, op=dist.ReduceOp.SUM)
            ce, hb, db = (float(x) for x in cc.tolist())
        e2e = {"value": ce / te, "unit": UNIT,
               "h2d_bytes_per_step": int(hb / args.steps),
               "d2h_bytes_per_step": int(db / args.steps),
               "timed": "restore(host pinned state -> HBM) + K coarse steps + snapshot(HBM -> host)"
                        + (", every rank its own pools, max over ranks" if world > 1 else "")}
        del sim2, snap, out

    # ---- CPU baseline (rank 0, N=1 only) -------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        workers = os.cpu_count() or 1
        v, t, desc, _ = run_cpu(args.config, 1, 0, workers, 64)
        cpu = {"value": v, "unit": UNIT, "cores": workers, "kind": "port",
               "sample": f"{desc}; 1 coarse step (all levels), oracle/ C+numpy port, {t:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: {pb.num_levels} levels, M={M}, "
                                   f"L1 {pb.coarse_nx}x{pb.coarse_ny}, ratios {pb.ratios_x}",
                       "patches_per_level": patches_per_level,
                       "cells_per_level": cells_per_level,
                       "parallelism": (f"SFC-sharded patches x{world} ({dist.get_backend()} shadow exchange)"
                                       if world > 1 else "single GPU"),
                       "l2": (f"inputs larger than L2 (device state {pool_bytes / 1e9:.2f} GB)" if pool_bytes > 126e6 else f"device state {pool_bytes / 1e9:.3f} GB fits in L2 (no flush)"),
                       "dt_policy": "reference: level-1 stable_dt, r_t subcycling",
                       **({"exchange_bytes_per_step_rank0": xbytes} if world > 1 else {}),
                       "host_ms_per_step": host_ms},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "traffic_over_algorithmic": traffic_ratio,
                         "traffic_source": "ncu --set full capture of one C4 level-3 launch "
                                           "(profiles/r02/step_traffic.json)",
                         "kernel": "mlamr_step (k_step) on the finest level",
                         "bytes_per_launch": int(np.mean(byts)) if byts else None,
                         "avg_launch_ms": 1e3 * float(np.mean(durs)) if durs else None,
                         "share_of_step": step_share, "peak_source": peak_kind},
            "kernels_roofline": kernels,
            "regrid_stress": stress,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk.summary(),
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    clk.stop()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-stress", action="store_true", help="skip the C5s regrid-stress measurement")
    ap.add_argument("--no-aux", action="store_true",
                    help="skip the auxiliary kernels' instrumented pass (kernels_roofline)")
    args = ap.parse_args()
    if args.impl == "reference":
        reference_arm(args)
    else:
        b200_arm(args)


if __name__ == "__main__":
    main()
