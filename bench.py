"""Benchmark of the hierarchical random-walker hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c4|c2|c3|c1]

One step = one full hierarchical random-walker segmentation of a synthetic
volume already resident in HBM: LOD pyramid, seed projection, coarsest-level
solve, upsample + brick-wise Jacobi-PCG solve of every finer level,
probabilities and labels of level 0 written to HBM.  `value` = level-0
voxels / second over all ranks (max-over-ranks device time).

Default workload = BASELINE.json config 4 (1024^3, 4 levels, 32^3 bricks),
the configuration the metric's 1/2/4/8-GPU scaling is quoted on; it fits one
B200.  Under torchrun (N > 1) the bricks of every level are sharded across
ranks (sharding.py) with an NCCL halo exchange between levels.

`--impl reference` times the CPU reference of the path (the float64 numpy
oracle, brick-parallel on all host cores; the reference package has no
random walker of its own) on a bounded sample of the same
workload and prints the same JSON line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "c4": dict(shape=(1024, 1024, 1024), brick=(32, 32, 32), levels=4,
               desc="config 4: 1024^3 f32 two-blob phantom + noise, 4-level hierarchy (1024/512/256/128), "
                    "32^3 bricks, seeds S1",
               sample=dict(shape=(256, 256, 256), levels=4)),
    "c2": dict(shape=(256, 256, 256), brick=(32, 32, 32), levels=2,
               desc="config 2: 256^3 f32 two-blob phantom + noise, 2-level hierarchy, 32^3 bricks, seeds S1",
               sample=dict(shape=(128, 128, 128), levels=2)),
    "c3": dict(shape=(16384, 16384), brick=(64, 64), levels=9,
               desc="config 3: 16384^2 f32 two-blob image + noise, 9-level hierarchy, 64^2 bricks, seeds S1",
               sample=dict(shape=(1024, 1024), levels=5)),
    "c5": dict(shape=(512, 512, 512), timesteps=16, brick=(32, 32, 32), levels=4,
               desc="config 5: 4-D series 512^3 x 16 timesteps (blobs shift along axis 1), per-timestep 4-level "
                    "hierarchy (512/256/128/64), 32^3 bricks, seeds S1; the series lives in pinned host memory "
                    "and streams through a bounded HBM store (one arena) holding 4 of its 16 timesteps",
               sample=dict(shape=(128, 128, 128), levels=2)),
    "c1": dict(shape=(64, 64, 64), brick=(32, 32, 32), levels=1,
               desc="config 1: 64^3 f32 two-blob phantom + noise, single level, seeds S1",
               sample=dict(shape=(64, 64, 64), levels=1)),
}
METRIC = "random-walker voxels/sec"
UNIT = "voxel/s"
BETA, WMIN, TOL = 100.0, 1e-6, 1e-6


# algorithmic bytes per unknown voxel per PCG iteration (fp32, forward-edge weights
# and the inverse diagonal stored): 3-D 56 B, 2-D 52 B.  (Our streaming kernels need 52 / 48 B: the
# Jacobi-scaled system has a unit diagonal.)
ALG_BYTES_PER_UNKNOWN_ITER = {3: 56, 2: 52}


STREAM_BYTES_PER_UNKNOWN_ITER = {3: 52, 2: 48}  # what the streaming CG passes move (csrc/rwb_solve.cu header)


def streaming_roofline(vol, seeds, brick, levels, cfg, peak, k1=2, k2=6):
    """The streaming CG passes (the solver of any brick shape the on-chip engines do not take) on the
    workload's level 0 with every brick active: device ms per iteration from k2 - k1 iterations,
    HBM rate from the passes' own algorithmic bytes.  Untimed with respect to the bench line."""
    import torch

    from paper_2509_26213_b200 import device
    from paper_2509_26213_b200.config import RWConfig

    vols = device.lod_chain(vol, brick, levels)
    if len(vols) < 2:  # one whole level: the cooperative / multigrid solvers, not the streaming passes
        return None
    k, brick_k = 0, brick
    bound = device.upsample(torch.full(vols[1].shape, 0.5, device=vol.device), vols[0].shape)
    ws = device.Workspace(vol.device)
    times = []
    st = None
    for iters in (k1, k2):
        c = RWConfig(beta=cfg.beta, min_weight=cfg.min_weight, tol=1e-30, max_iter=iters, check_every=iters,
                     resident=False)
        device.solve_level(vols[k], seeds, brick_k, bound, c, workspace=ws)  # graph capture
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, st = device.solve_level(vols[k], seeds, brick_k, bound, c, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    per = (times[1] - times[0]) / (k2 - k1)
    nd = len(vol.shape)
    b = STREAM_BYTES_PER_UNKNOWN_ITER[nd]
    gbs = b * st["unknowns"] / (per / 1e3) / 1e9
    del ws
    return {"level": k, "shape": list(vols[k].shape), "brick": list(brick_k), "path": st["path"],
            "kernels": "cg_pass1_stg_kernel + cg_pass2_vec_kernel" if nd == 3 else
                       "cg_pass1_brick2d_kernel + cg_pass2_vec_kernel",
            "ms_per_iteration": per, "unknowns": st["unknowns"], "bytes_per_unknown_iteration": b,
            "achieved": gbs, "peak": peak, "frac": gbs / peak,
            "note": f"every brick active (tol 1e-30), {k2}-{k1} iterations differenced; bytes = what the two "
                    "passes read and write per unknown (r, p, w'x, w'y, w'z in / p, q out; y, r, p, q in / y, r "
                    "out), the north star's fused-CG HBM figure"}


def load_traffic(config, level_key):
    """The ncu capture of the dominant kernel (profiles/rNN_traffic.json, newest round first,
    written by tools/ncu_traffic.py): per-level DRAM bytes and on-chip utilisation, or None."""
    import glob

    prof = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles")
    files = sorted(glob.glob(os.path.join(prof, "r*_traffic.json")),
                   key=lambda f: int(os.path.basename(f)[1:].split("_")[0]), reverse=True)
    for path in files:
        try:
            with open(path) as f:
                got = json.load(f).get(config, {}).get(level_key)
        except (OSError, ValueError):
            continue
        if isinstance(got, dict):
            return dict(got, file=os.path.relpath(path, os.path.dirname(prof)))
        if got is not None:
            return {"bytes_per_level": got, "file": os.path.relpath(path, os.path.dirname(prof))}
    return None


def load_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        period = int(os.environ.get("RWB_BENCH_CLOCK_MS", "200"))  # diagnostics: 0 = no sampling
        if period <= 0:
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", str(period)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference (oracle) on a bounded sample


def cpu_reference_sample(wl, steps=1, warmup=0, inputs=None):
    """The CPU reference (float64 numpy oracle on the host's cores) for a workload, by the
    BASELINE.md §4 plan: config 1 timed fully; larger configs extrapolated from a per-step sample
    (oracle/cpu_baseline.py: slab LOD, the whole coarsest solve, brick chains per finer level).
    `inputs` = (volume, seeds) numpy arrays of the workload (generated here when None).
    Returns (level-0 voxels, per-step seconds, cores, sample description, per-part seconds)."""
    import numpy as np

    from oracle import cpu_baseline as cbl
    from oracle import rw as orw
    from paper_2509_26213_b200 import synthetic

    params = orw.RWParams(beta=BETA, min_weight=WMIN, tol=TOL, max_iter=10_000)
    shape = tuple(wl["shape"])
    cores = len(os.sched_getaffinity(0))
    if wl is WORKLOADS["c1"]:
        vol = synthetic.phantom(shape)
        seeds = synthetic.seeds(shape, "S1")
        times = []
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            orw.hierarchical_random_walker(vol, seeds, wl["brick"], wl["levels"], params, threads=1)
            if i >= warmup:
                times.append(time.perf_counter() - t0)
        return (math.prod(shape), times, 1, "the full configuration (64^3, one level), float64 numpy oracle, "
                "1 thread", None)
    if inputs is None:
        slab = max(1, (1 << 24) // math.prod(shape[1:]))
        vol = np.empty(shape, np.float32)
        seeds = np.empty(shape, np.uint8)
        if "timesteps" in wl:
            synthetic.series_timestep(shape, 0, wl["timesteps"], slab=slab, out=vol)
            synthetic.seeds_streamed(shape, "S1", t=0, steps=wl["timesteps"], slab=slab, out=seeds)
        else:
            synthetic.phantom_streamed(shape, slab=slab, out=vol)
            synthetic.seeds_streamed(shape, "S1", slab=slab, out=seeds)
    else:
        vol, seeds = inputs
    base = cbl.C4Baseline(vol, seeds, wl["brick"], wl["levels"], params, cores=cores, chains=cores,
                          slab_planes=min(128, shape[0]))
    times, parts = [], None
    try:
        for i in range(warmup + steps):
            total, parts = base.step()
            if i >= warmup:
                times.append(total)
    finally:
        base.close()
    nd = len(shape)
    per = 2 ** nd
    sample = (f"extrapolated (BASELINE.md §4): the real {'x'.join(map(str, shape))} input and its full "
              f"{wl['levels']}-level pyramid; per step, timed on {cores} threads: the LOD + seed projection of a "
              f"{min(128, shape[0])}-plane level-0 slab (scaled by planes), {base.top_sample} iterations of the "
              f"coarsest {'x'.join(map(str, base.shapes[-1]))} Jacobi-PCG scaled to its {base.top_iterations} "
              f"(the full solve, timed once at setup: {base.top_full_seconds:.1f} s), the prolongation (scaled by "
              f"voxels), and {cores} brick chains ({per} real bricks per finer level each, true Dirichlet halos) "
              f"scaled by brick count; float64 numpy oracle")
    if "timesteps" in wl:
        sample += f"; one timestep of the {wl['timesteps']}-step series (the same per-voxel rate for all)"
    return math.prod(shape), times, cores, sample, parts


def host_inputs(shape, t=None, steps=1):
    """Pinned host volume + seeds from the 8(d) generator (timestep t of the 4-D series when given)."""
    import torch

    from paper_2509_26213_b200 import synthetic

    slab = max(1, (1 << 24) // math.prod(shape[1:]))
    vol_h = torch.empty(shape, dtype=torch.float32, pin_memory=True)
    seeds_h = torch.empty(shape, dtype=torch.uint8, pin_memory=True)
    if t is None:
        synthetic.phantom_streamed(shape, slab=slab, out=vol_h.numpy())
        synthetic.seeds_streamed(shape, "S1", slab=slab, out=seeds_h.numpy())
    else:
        synthetic.series_timestep(shape, t, steps, slab=slab, out=vol_h.numpy())
        synthetic.seeds_streamed(shape, "S1", t=t, steps=steps, slab=slab, out=seeds_h.numpy())
    return vol_h, seeds_h


def run_series(args, wl, rank, world):
    """Config 5: a step = the whole 4-D series through api.segment_series (streamed from host)."""
    import torch

    import __graft_entry__ as entry

    entry.build()
    from paper_2509_26213_b200 import _native, api, device, synthetic
    from paper_2509_26213_b200.config import RWConfig

    local = local_device()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = _native.lib()
    cfg = RWConfig(beta=BETA, min_weight=WMIN, tol=TOL, max_iter=10_000, check_every=args.check_every)
    shape, brick, levels, n_t = wl["shape"], wl["brick"], wl["levels"], wl["timesteps"]
    full = (n_t,) + tuple(shape)
    # N ranks: timesteps dealt round-robin (independent problems, no exchange); each rank
    # holds only its own timesteps, in pinned host memory
    mine = list(range(rank, n_t, world))
    local_shape = (len(mine),) + tuple(shape)
    vol_h = torch.empty(local_shape, dtype=torch.float32, pin_memory=True)
    sd_h = torch.empty(local_shape, dtype=torch.uint8, pin_memory=True)
    slab = max(1, (1 << 24) // math.prod(shape[1:]))
    for i, t in enumerate(mine):  # 8(d) generator per timestep, kept in pinned host memory (untimed)
        synthetic.series_timestep(shape, t, n_t, slab=slab, out=vol_h[i].numpy())
        synthetic.seeds_streamed(shape, "S1", t=t, steps=n_t, slab=slab, out=sd_h[i].numpy())
    outs = (torch.empty(local_shape, dtype=torch.float32, pin_memory=True),
            torch.empty(local_shape, dtype=torch.uint8, pin_memory=True))
    ws = device.Workspace(dev)
    # the timesteps stream through a bounded HBM store (one arena) holding 4 of them, far below
    # the series' working set: every step uploads every timestep into it, evicting LRU-first
    from paper_2509_26213_b200.store import DeviceStore

    per_t = 5 * math.prod(shape)
    store = DeviceStore(4 * per_t + (1 << 20), dev)
    warm = max(1, min(args.warmup, 3))
    for _ in range(warm):
        api.segment_many([(vol_h[t], sd_h[t]) for t in range(min(2, len(mine)))], brick, levels, cfg,
                         outputs=[(outs[0][t], outs[1][t]) for t in range(min(2, len(mine)))], workspace=ws)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = lib.rwb_kernel_launches()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            api.segment_series(vol_h, sd_h, brick, levels, cfg, outputs=outs, workspace=ws, store=store)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = lib.rwb_kernel_launches() - launches0
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        tm = torch.tensor([ms], dtype=torch.float64, device=dev)
        all_reduce_(tm, dist.ReduceOp.MAX)
        ms = float(tm.item())
    nvox = math.prod(full)
    # kernel-level view: one timestep device-resident
    v0 = vol_h[0].to(dev)
    s0 = sd_h[0].to(dev)
    device.hierarchical_random_walker(v0, s0, brick, levels, cfg, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    res = device.hierarchical_random_walker(v0, s0, brick, levels, cfg, workspace=ws)
    e1.record(stream)
    torch.cuda.synchronize()
    t_ms = e0.elapsed_time(e1)
    peak, peak_src = load_peak()
    alg_b = ALG_BYTES_PER_UNKNOWN_ITER[3]
    lv = max((s for s in res.stats if s), key=lambda s: s["cg_ms"])
    gbs = alg_b * lv["unknown_iterations"] / (lv["cg_ms"] / 1e3) / 1e9
    comm = comm_info(world)  # collective: every rank
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n, times, cores, sample, parts = cpu_reference_sample(wl, steps=1)
        cpu = {"value": n / times[0], "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
               "seconds": parts}
    if rank == 0:
        line = {
            "metric": METRIC, "value": nvox / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": warm, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic: SURVEY.md 8(d) 4-D series (synthetic.series_timestep: blobs shifted along axis 1, "
                    "numpy noise seed 0xC0FFEE + t), held in pinned host memory",
            "config": {"workload": wl["desc"], "size": list(full), "brick": list(brick), "levels": levels,
                       "beta": BETA, "min_weight": WMIN, "tol": TOL,
                       "parallelism": f"timesteps round-robin over {world} GPUs" if world > 1 else "1 GPU (timestep stream)",
                       "l2": "every timestep uploaded from host (512 MiB f32) > 126 MB L2",
                       "device_store": {"capacity_bytes": store.capacity, "series_input_bytes": per_t * len(mine),
                                        "peak_occupancy": store.peak_occupancy, "evictions": store.evictions,
                                        "hits": store.hits, "misses": store.misses}},
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                         "traffic": None, "peak_source": peak_src,
                         "kernel": f"level-{res.stats.index(lv)} solve of one timestep (path {lv['path']}), "
                                   f"{alg_b} B per unknown-iteration (SURVEY.md 8(d))",
                         "timestep_device_resident_ms": t_ms},
            "cpu_baseline": cpu,
            "e2e": {"value": nvox / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
                    "h2d_bytes_per_step": nvox * 5, "d2h_bytes_per_step": nvox * 5,
                    "api": "paper_2509_26213_b200.api.segment_series (host series streamed through "
                           "segment_many; the value above is this end-to-end number)"},
            "clocks": clocks.summary(), "gpu_launches": int(launches), "comm": comm,
            "levels": [dict(st, level=k) for k, st in enumerate(res.stats) if st is not None],
        }
        print(json.dumps(line), flush=True)
    return 0


def run_reference(args, wl, rank):
    if rank != 0:
        return 0
    n, times, cores, sample, parts = cpu_reference_sample(wl, args.steps, args.warmup)
    total = sum(times)
    value = n * len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["desc"], "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                         "seconds_last_step": parts},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our path


def run_ours(args, wl, rank, world):
    import numpy as np
    import torch
    import torch.distributed as dist

    import __graft_entry__ as entry

    entry.build()
    from paper_2509_26213_b200 import _native, api, device, sharding, synthetic
    from paper_2509_26213_b200.config import RWConfig

    local = local_device()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = _native.lib()
    cfg = RWConfig(beta=BETA, min_weight=WMIN, tol=TOL, max_iter=10_000, check_every=args.check_every)
    shape, brick, levels = wl["shape"], wl["brick"], wl["levels"]
    nvox = math.prod(shape)
    # SURVEY.md 8(d) inputs: the numpy generator (default_rng(0xC0FFEE)), streamed slab by slab into
    # pinned host memory (bit-identical to synthetic.phantom; the inputs the parity tests pin,
    # tests/test_bench_configs.py), then made resident in HBM (untimed)
    vol_h, seeds_h = host_inputs(shape)
    ws = device.Workspace(dev)
    plan = sharding.ShardPlan.build(shape, brick, levels, rank, world) if world > 1 else None
    if plan is not None:  # each rank holds only its level-0 slab (sharding.py)
        a, b = plan.lod_slab(0)
        vol_h, seeds_h = vol_h[a:b].clone().pin_memory(), seeds_h[a:b].clone().pin_memory()
    vol = vol_h.to(dev)
    seeds = seeds_h.to(dev)
    cpu_inputs = (vol_h.numpy(), seeds_h.numpy()) if world == 1 else None
    level_voxels = [math.prod(s) for s in sharding.level_shapes(shape, levels)]

    def step():
        if plan is None:
            return device.hierarchical_random_walker(vol, seeds, brick, levels, cfg, workspace=ws)
        return sharding.hierarchical_random_walker_sharded(vol, seeds, plan, cfg, workspace=ws)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        res = step()
    torch.cuda.synchronize()
    barrier()

    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = lib.rwb_kernel_launches()
    # per level solve (one resident / cooperative launch, or the streaming CG launches of a level):
    # device ms and SURVEY.md 8(d) algorithmic bytes = 56 B (3-D; 52 B 2-D) per unknown voxel per
    # PCG iteration, counted exactly on the device (sum over bricks of unknowns x iterations)
    acc = {}
    alg_b = ALG_BYTES_PER_UNKNOWN_ITER[len(shape)]
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            res = step()
            for k, st in enumerate(res.stats):
                if st is None:
                    continue
                a = acc.setdefault(k, {"ms": 0.0, "alg_bytes": 0.0, "unknown_iterations": 0, "path": st["path"],
                                       "voxels": level_voxels[k], "brick_iterations": 0})
                a["brick_iterations"] += st["iterations_sum"]
                a["ms"] += st["cg_ms"]
                a["alg_bytes"] += alg_b * st["unknown_iterations"]
                a["unknown_iterations"] += st["unknown_iterations"]
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = lib.rwb_kernel_launches() - launches0
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        all_reduce_(t, dist.ReduceOp.MAX)
    ms_max = float(t.item())
    per_level = [dict(st, level=k, shape=list(sharding.level_shapes(shape, levels)[k]))
                 for k, st in enumerate(res.stats) if st is not None]
    shard_info = None
    if plan is not None:
        shard_info = {"lod_slabs_level0": plan.lod[0], "solve_rows": res.solve_rows[:-1],
                      "result_planes": [res.z0, res.z1]}

    # end to end through the public API with pinned host buffers
    e2e = None
    if world > 1 and not args.no_e2e:
        # every rank: upload its input slab, run its part of the hierarchy, download its result
        # planes (probabilities + labels), device-timed, max over ranks
        out_p = torch.empty(tuple(res.prob.shape), dtype=torch.float32, pin_memory=True)
        out_l = torch.empty(tuple(res.prob.shape), dtype=torch.uint8, pin_memory=True)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            vd = vol_h.to(dev, non_blocking=True)
            sdd = seeds_h.to(dev, non_blocking=True)
            r = sharding.hierarchical_random_walker_sharded(vd, sdd, plan, cfg, workspace=ws)
            out_p.copy_(r.prob, non_blocking=True)
            out_l.copy_(r.labels, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        all_reduce_(te, dist.ReduceOp.MAX)
        e_ms = float(te.item()) / args.steps
        hb = torch.tensor([vol_h.numel() * 5, out_p.numel() * 5], dtype=torch.float64, device=dev)
        all_reduce_(hb)
        e2e = {"value": nvox / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(hb[0].item()), "d2h_bytes_per_step": int(hb[1].item()),
               "api": "paper_2509_26213_b200.sharding.hierarchical_random_walker_sharded: every rank uploads its "
                      "level-0 input slab from pinned host memory and downloads its result planes each step "
                      "(bytes summed over ranks; time = max over ranks)"}
    if world == 1 and not args.no_e2e:
        outs = [(torch.empty(shape, dtype=torch.float32, pin_memory=True),
                 torch.empty(shape, dtype=torch.uint8, pin_memory=True)) for _ in range(2)]
        # single call (latency): upload, segment, download in sequence
        api.segment(vol_h, seeds_h, brick, levels, cfg, out_prob=outs[0][0], out_labels=outs[0][1], workspace=ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        api.segment(vol_h, seeds_h, brick, levels, cfg, out_prob=outs[0][0], out_labels=outs[0][1], workspace=ws)
        e1.record(stream)
        torch.cuda.synchronize()
        lat_ms = e0.elapsed_time(e1)
        # K volumes through the streaming API (throughput): every step still uploads its
        # inputs and downloads its result, overlapped with the neighbouring steps' compute
        api.segment_many([(vol_h, seeds_h)] * 2, brick, levels, cfg, outputs=outs, workspace=ws,
                         cyclic_outputs=True)
        torch.cuda.synchronize()
        e0.record(stream)
        api.segment_many([(vol_h, seeds_h)] * args.steps, brick, levels, cfg, outputs=outs, workspace=ws,
                         cyclic_outputs=True)
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / args.steps
        e2e = {"value": nvox / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": vol_h.numel() * 4 + seeds_h.numel(),
               "d2h_bytes_per_step": outs[0][0].numel() * 4 + outs[0][1].numel(),
               "api": "paper_2509_26213_b200.api.segment_many (pinned host in/out; step k+1's upload and "
                      "step k-1's download overlap step k's compute on their own streams)",
               "latency_ms_single_call": lat_ms,
               "latency_api": "paper_2509_26213_b200.api.segment (upload, segment, download in sequence)"}
        del outs

    peak, peak_src = load_peak()
    path_name = {0: "streaming cg_pass1/cg_pass2", 1: "resident3d_q4_kernel" if len(wl["shape"]) == 3 else
                 "resident2d_kernel", 2: "coop_cg_kernel", 3: "mgcg_kernel"}
    kernels = {}
    for k, a in sorted(acc.items()):
        if a["ms"] <= 0:
            continue
        gbs = a["alg_bytes"] / (a["ms"] / 1e3) / 1e9
        kernels[f"level{k}"] = {
            "kernel": path_name.get(a["path"], "?"), "ms_per_step": a["ms"] / args.steps,
            "share_of_step": a["ms"] / ms_max, "achieved_gbs": gbs, "frac": gbs / peak,
            "unknown_iterations_per_step": a["unknown_iterations"] // args.steps,
            "brick_iterations_per_step": a["brick_iterations"] // args.steps,
        }
    dom = max(kernels, key=lambda n: kernels[n]["ms_per_step"])
    dk = kernels[dom]
    prof = load_traffic(args.config, dom)
    traffic = prof["bytes_per_level"] if prof else None
    clk = clocks.summary()
    onchip = None
    need = ("grid_size", "cluster_dim", "issue_active_pct", "fma_pipe_pct", "bytes_per_voxel")
    if prof and all(k in prof for k in need) and acc.get(int(dom[5:]), {}).get("path") == 1 and clk.get("sm_mhz"):
        # the resident engine's real limit: cycles per brick iteration of one cluster (live), beside
        # the ncu issue / FMA-pipe activity of the same kernel and the HBM bytes it actually moves
        clusters = prof["grid_size"] // max(1, prof["cluster_dim"])
        per_step_ms = dk["ms_per_step"]
        cyc = per_step_ms * 1e-3 * clk["sm_mhz"] * 1e6 * clusters / max(1, dk["brick_iterations_per_step"])
        actual_gbs = traffic / (per_step_ms / 1e3) / 1e9
        onchip = {"cycles_per_brick_iteration": cyc, "clusters": clusters, "sm_mhz": clk["sm_mhz"],
                  "issue_active_pct": prof["issue_active_pct"], "fma_pipe_pct": prof["fma_pipe_pct"],
                  "hbm_bytes_per_voxel": prof["bytes_per_voxel"], "hbm_gbs_actual": actual_gbs,
                  "hbm_frac_actual": actual_gbs / peak, "profile": prof.get("file"),
                  "profile_commit": prof.get("commit")}
    roofline = {"bound": "hbm", "achieved": dk["achieved_gbs"], "peak": peak, "unit": "GB/s", "frac": dk["frac"],
                "traffic": traffic, "onchip": onchip,
                "kernel": f"{dk['kernel']} ({dom}: the level with the largest solve time; its launches)",
                "algorithmic_bytes": f"{alg_b} B per unknown voxel per PCG iteration (SURVEY.md 8(d)) x "
                                     f"{dk['unknown_iterations_per_step']} unknown-iterations per launch",
                "peak_source": peak_src,
                "note": ("frac > 1: the brick-resident engine keeps every CG vector of a brick on chip (registers, "
                         "TMEM and SMEM of a 4-CTA cluster), so per-iteration traffic never reaches HBM; the HBM roofline of "
                         "the streaming algorithm (the 8(d) bytes) is beaten, and the kernel is bound by the "
                         "latency of its per-iteration cluster reduction instead (achieved counts 56 B per "
                         "EXECUTED unknown-iteration: the default coarse-corrected engine runs a third fewer "
                         "iterations than Jacobi-PCG for the same stop rule, so a faster solve reports a lower "
                         "work rate); onchip = live cycles per brick "
                         "iteration per cluster, with the ncu issue / FMA-pipe activity and the bytes the kernel "
                         "really moves (hbm_frac_actual); traffic = ncu DRAM bytes of the level's launches, from "
                         "the profile named in onchip.profile"),
                "kernels": kernels}
    if rank == 0 and world == 1 and os.environ.get("RWB_BENCH_NO_STREAMING") != "1":
        roofline["streaming_cg"] = streaming_roofline(vol, seeds, brick, levels, cfg, peak)

    comm = comm_info(world)  # collective: every rank
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n, times, cores, sample, parts = cpu_reference_sample(wl, steps=1, inputs=cpu_inputs)
        cpu = {"value": n / times[0], "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
               "seconds": parts}

    if rank == 0:
        line = {
            "metric": METRIC, "value": nvox * args.steps / (ms_max / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic: SURVEY.md 8(d) two-blob phantom, numpy default_rng(0xC0FFEE) noise "
                                    "(synthetic.phantom_streamed), seeds S1",
            "config": {"workload": wl["desc"], "size": list(shape), "brick": list(brick), "levels": levels,
                       "beta": BETA, "min_weight": WMIN, "tol": TOL, "parallelism": f"bricks sharded x{world}"
                       if world > 1 else "1 GPU",
                       "l2": f"inputs {nvox * 5 / 2**30:.1f} GiB (f32 volume + u8 seeds) > 126 MB L2; no flush"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk,
            "gpu_launches": int(launches),
            "comm": comm,
            "levels": per_level,
        }
        if shard_info is not None:
            line["sharding"] = shard_info
        print(json.dumps(line), flush=True)
    return 0


def _free_port() -> int:
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """`--gpus N` (N > 1) without a torchrun environment: relaunch this command as N ranks, one
    process per GPU, under torch.distributed.run on 127.0.0.1; rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.run(cmd, env=env).returncode


def all_reduce_(t, op=None):
    """dist.all_reduce in place; a CUDA tensor goes through host memory when the backend is not
    NCCL (the RWB_BENCH_SHARE_GPU gloo dry run)."""
    import torch.distributed as dist

    op = dist.ReduceOp.SUM if op is None else op
    if t.is_cuda and dist.get_backend() != "nccl":
        h = t.cpu()
        dist.all_reduce(h, op=op)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op)
    return t


def local_device() -> int:
    """This rank's GPU: LOCAL_RANK, or 0 for every rank with RWB_BENCH_SHARE_GPU=1 (a multi-rank
    dry run of the sharded path on a one-GPU box, over gloo; never a measurement)."""
    return 0 if os.environ.get("RWB_BENCH_SHARE_GPU") == "1" else int(os.environ.get("LOCAL_RANK", 0))


def init_ranks(world: int):
    """Process group of the N ranks (NCCL on GPUs; gloo where there is no CUDA device)."""
    import torch
    import torch.distributed as dist

    if world <= 1 or dist.is_initialized():
        return
    if torch.cuda.is_available():
        torch.cuda.set_device(local_device())
        if os.environ.get("RWB_BENCH_SHARE_GPU") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_device()))
    else:
        dist.init_process_group("gloo")


def comm_info(world: int) -> dict:
    """Rank count the communicator actually has, and the GPU each rank drives (all-gathered)."""
    import torch

    if world <= 1:
        dev = torch.cuda.current_device() if torch.cuda.is_available() else -1
        return {"backend": None, "nranks": 1, "devices": [dev]}
    import torch.distributed as dist

    cuda = torch.cuda.is_available()
    mine = torch.tensor([torch.cuda.current_device() if cuda else -1], dtype=torch.int64,
                        device="cuda" if cuda and dist.get_backend() == "nccl" else "cpu")
    got = [torch.zeros_like(mine) for _ in range(dist.get_world_size())]
    dist.all_gather(got, mine)
    return {"backend": dist.get_backend(), "nranks": dist.get_world_size(), "devices": [int(t.item()) for t in got]}


def run_launch_probe(args, rank, world):
    """`--launch-probe`: start the ranks exactly as a measured run does (spawned or torchrun),
    exchange once over the communicator and print the line's launch fields (no kernels; runs on
    CPU with gloo, which is how the test suite checks `--gpus N`)."""
    import torch

    init_ranks(world)
    info = comm_info(world)
    if world > 1:
        import torch.distributed as dist

        one = torch.ones(1, device="cuda" if torch.cuda.is_available() else "cpu")
        all_reduce_(one)
        info["all_reduce_ok"] = int(one.item()) == world
    if rank == 0:
        print(json.dumps({"launch_probe": True, "n_gpus": world, "requested_gpus": args.gpus, "comm": info}),
              flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(WORKLOADS), default="c4")
    ap.add_argument("--check-every", type=int, default=16)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--launch-probe", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.launch_probe:
        return run_launch_probe(args, rank, world)
    wl = WORKLOADS[args.config]
    if args.impl == "reference":
        return run_reference(args, wl, rank)
    init_ranks(world)
    try:
        if "timesteps" in wl:
            return run_series(args, wl, rank, world)
        return run_ours(args, wl, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
