"""BEV-pool benchmark (BASELINE.json metric) -- one JSON line on stdout.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (configs[1], SURVEY.md §8 "S"): nuScenes camera stream, 6 cameras x
32x88 features, D=118 (1-60 m @ 0.5 m), C=80, 360x360 BEV grid @ 0.3 m,
batch 1, cached-interval forward.  A step is one reference-API forward
``pool_interval(features, dist, cache, grid, SUM)`` through the pixel-column
tiled path (csrc/tile.cu: tile reduction + per-cell combine into the map),
inputs resident in HBM, L2 flushed (512 MiB write) between steps.  value =
frustum points/s over all ranks (each rank pools its own sample: weak
scaling, no collective in the loop; NCCL only gathers the timings).  e2e =
the same step through PoolPlan.run_frames with host buffers (pinned H2D of
features + dist, D2H of the BEV map) in the timed region.  N=1 also reports
cpu_baseline (the reference's own pool_interval from baseline/_ref on all
host threads; the oracle's C port only if that is missing) and the other
configurations as "variants".

``--impl reference`` times the reference's own CPU pool_interval (installed
unmodified into baseline/_ref; numba/OpenMP over all host cores; the
oracle's C port when absent) on the same config; under torchrun only rank 0
runs it.
"""

from __future__ import annotations

import argparse
import functools
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "bev_pool_points_per_sec"
UNIT = "points/s"
CONFIG_NAME = "S"
FLUSH_BYTES = 512 << 20
KERNEL_KEYS = ("tile_pool_kernel", "tile_finalize_kernel")
# the tiled path: tile reduction (phase 1) + per-cell combine into the map (phase 2)
LAUNCHES_PER_STEP = 2
# pure L2 gather of the S-config rows in rank order (scripts/gather_mlp_bench.cu,
# profiles/r01/gather_mlp_bench.txt)
L2_GATHER_CEILING_GBPS = 13610.0


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="S", choices=["S", "F", "B", "H"],
                    help="S: cached forward, 1 sample/GPU (the headline); F: the fused bf16 "
                         "lift+pool forward from logits and context, 1 sample/GPU; B: training "
                         "step (forward + backward), batch 4/GPU; H: high-res frame with the "
                         "association rebuilt every step, 1 sample/GPU")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def config_dict(spec):
    """The workload, identical in both arms (the driver compares them)."""
    f, g = spec.frustum, spec.grid
    return {"workload": "nuScenes camera stream (configs[1]): cached-interval forward",
            "cameras": spec.n_cameras, "feature_hw": [f.height, f.width],
            "depth_bins": f.depth_bins, "channels": spec.channels, "grid": [g.nx, g.ny],
            "cell_m": g.r, "batch_per_gpu": 1, "points_per_sample": spec.n_points,
            "reducer": "sum"}


# ---------------------------------------------------------------------------
# CPU reference arm
# ---------------------------------------------------------------------------

def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


REF_DIR = os.path.join(ROOT, "baseline", "_ref")

# Runs in a fresh interpreter: the reference sizes its OpenMP pool at import
# (pkg/src/bevpool/_threads.py:32-37), and OpenBLAS spin threads starve it
# unless OPENBLAS_NUM_THREADS=1.
_REF_SNIPPET = r"""
import json, os, sys, time
sys.path.insert(0, os.environ["BVP_REF_DIR"])
import numpy as np
import bevpool as ref
from bevpool.bevgrid import BevGridSpec
from bevpool.geometry import FrustumSpec
reps, warm, max_s = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
spec = ref.WorkloadSpec(6, FrustumSpec(32, 88, 1.0, 0.5, 118),
                        BevGridSpec(-54.0, 54.0, -54.0, 54.0, -10.0, 10.0, 0.3), 80, 0)
rig, feats, logits, grid = ref.gen_workload(spec)
cache = ref.build_cache(rig, spec.frustum, grid)
dist = ref.normalize_depth(logits)
for _ in range(warm):
    ref.pool_interval(feats, dist, cache, grid, ref.Reducer.SUM)
ts = []
t_start = time.perf_counter()
while len(ts) < reps:
    t0 = time.perf_counter()
    ref.pool_interval(feats, dist, cache, grid, ref.Reducer.SUM)
    ts.append(time.perf_counter() - t0)
    if time.perf_counter() - t_start > max_s and len(ts) >= 3:
        break
print(json.dumps({"times": ts, "threads": ref.get_parallelism()}))
"""


def time_cpu_reference(spec, max_seconds, min_reps=3, max_reps=200, warmup=1):
    """The reference's own pool_interval (pkg/src/bevpool/pooling.py:206-221,
    numba + OpenMP) from baseline/_ref on all host threads, in a subprocess.
    Falls back to the oracle's C port of it when the reference is not
    installed.  Returns (per-step seconds, threads, kind)."""
    if os.path.isdir(os.path.join(REF_DIR, "bevpool")):
        env = dict(os.environ, BVP_REF_DIR=REF_DIR, OPENBLAS_NUM_THREADS="1",
                   BEVPOOL_THREADS=str(cpu_threads()), NUMBA_NUM_THREADS=str(cpu_threads()),
                   NUMBA_CACHE_DIR=os.environ.get("NUMBA_CACHE_DIR", "/tmp/bvp_numba_cache"))
        res = subprocess.run([sys.executable, "-c", _REF_SNIPPET, str(max_reps), str(warmup),
                              str(max_seconds)], capture_output=True, text=True, env=env,
                             timeout=min(3600.0, max(600.0, 10 * max_seconds)))
        if res.returncode == 0:
            out = json.loads(res.stdout.strip().splitlines()[-1])
            return out["times"], out["threads"], "reference"
        print(f"reference arm failed, using the oracle port: {res.stderr[-400:]}",
              file=sys.stderr)
    from oracle import oracle as o

    lib = o.lib()
    lib.oracle_set_threads(cpu_threads())
    cfg = o.CONFIGS[CONFIG_NAME]
    cache = o.build_cache(cfg)
    f, lg = o.gen_inputs(cfg.n_cameras, cfg.channels, cfg.height, cfg.width, cfg.depth_bins, 0)
    dist = o.normalize_depth(lg)
    args = (f, dist, cache["ranks"], cache["interval_starts"], cache["interval_cells"],
            cfg.n_cells, "sum")
    for _ in range(warmup):
        o.pool_interval(*args)
    times = []
    t_start = time.perf_counter()
    while len(times) < max_reps:
        t0 = time.perf_counter()
        o.pool_interval(*args)
        times.append(time.perf_counter() - t0)
        if len(times) >= min_reps and time.perf_counter() - t_start > max_seconds:
            break
    return times, lib.oracle_max_threads(), "port"


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2205_13542_b200.workload import CONFIGS

    spec = CONFIGS[CONFIG_NAME]
    reps = max(1, args.steps)
    times, threads, kind = time_cpu_reference(spec, max_seconds=1e9, min_reps=reps,
                                              max_reps=reps, warmup=max(1, args.warmup))
    total = sum(times)
    value = spec.n_points * len(times) / total
    what = ("the reference's pool_interval (baseline/_ref, numba/OpenMP)" if kind == "reference"
            else "the oracle's C port of the reference's pool_interval (OpenMP)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 in / f64 accumulate", "data": "synthetic",
        "config": config_dict(spec),
        "impl_detail": what,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{len(times)} full nuScenes-shape pool_interval steps ({what}, "
                                   "incl. its NHWC transposes)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU helpers
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self, busy_only=True):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:  # pragma: no cover
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
            except ValueError:
                continue
            sm.append(s)
            smax = m
            for nm, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        busy = [s for s in sm if s > 0.5 * max(sm)] if busy_only else sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": smax,
                "samples": len(sm), "reasons": sorted(reasons)}


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel_keys):
    """dram read+write bytes per step of the headline kernels (summed) from
    the committed ncu --set full summary, if present."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            js = json.load(fh)
        vals = [js.get(k, {}).get("dram_bytes") for k in kernel_keys]
        return None if any(v is None for v in vals) else float(sum(vals))
    except (OSError, ValueError):
        return None


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as tdist

    import paper_2205_13542_b200 as bp
    from paper_2205_13542_b200.bevgrid import ptr, stream_ptr  # noqa: F401

    from paper_2205_13542_b200.shard import (gather_maps, gather_scalars, max_over_ranks,
                                             sample_seeds)

    rank, world, local = dist_env()
    # one process per GPU; BVP_BENCH_BACKEND=gloo + more ranks than GPUs is
    # only for exercising the multi-rank path on a single-GPU box
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        backend = os.environ.get("BVP_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            tdist.init_process_group(backend)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.config != "S":
        run_config_bh(args, bp, torch, tdist, dev, rank, world, local)
        return
    spec = bp.CONFIGS[CONFIG_NAME]
    f = spec.frustum
    P = spec.n_points

    # ---- inputs: this rank's sample (seed = rank), resident in HBM -------
    (seed,) = sample_seeds(world, rank, world)  # one sample per GPU, seed = sample index
    rig, feats_np, logits_np, grid = bp.gen_workload(
        bp.WorkloadSpec(spec.n_cameras, f, spec.grid, spec.channels, seed))
    cache = bp.build_cache(rig, f, grid, device=dev)
    feats = torch.from_numpy(feats_np).to(dev).view(1, *feats_np.shape)
    dist = bp.normalize_depth(torch.from_numpy(logits_np).to(dev)).view(1, *logits_np.shape)
    plan = bp.PoolPlan(cache, grid, spec.n_cameras, spec.channels, f.height, f.width,
                       f.depth_bins, 1, bp.Reducer.SUM, False, dev)
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(max(3, args.warmup)):
        flush.zero_()
        plan.run(feats, dist)
    K = args.steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize(dev)
    # the step: PoolPlan.run as one CUDA graph (the tiled path: tile
    # reduction, then the per-cell combine into the map); one host call per
    # frame
    assert plan.tiled, "the headline step is the tiled path"
    g_s = plan.graphed(plan.run, feats, dist)
    g_s.replay()
    for k in range(K):
        flush.zero_()
        ev[k][0].record(stream)
        g_s.replay()
        ev[k][2].record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        tdist.barrier()
    step_ms = [e[0].elapsed_time(e[2]) for e in ev]
    # per kernel: the same two launches as two graphs with an event between
    g_1 = plan.graphed(functools.partial(plan.phase, which=1), feats, dist)
    g_2 = plan.graphed(functools.partial(plan.phase, which=2), feats, dist)
    for k in range(K):
        flush.zero_()
        ev[k][0].record(stream)
        g_1.replay()
        ev[k][1].record(stream)
        g_2.replay()
        ev[k][2].record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        tdist.barrier()
    p1_ms = [e[0].elapsed_time(e[1]) for e in ev]
    p2_ms = [e[1].elapsed_time(e[2]) for e in ev]
    split_ms = [e[0].elapsed_time(e[2]) for e in ev]
    tot_ms = sum(step_ms)
    # e2e: host buffers (pinned) through the public serving API
    # (PoolPlan.run_frames): every step copies its features + dist H2D,
    # pools, and copies the BEV map D2H; consecutive frames overlap their
    # copies (two device buffer sets, separate copy streams); wall clock
    # over all K frames after a synchronize.
    h_feats = torch.from_numpy(feats_np).pin_memory()
    h_dist = dist.cpu().pin_memory()
    h_out = [torch.empty(tuple(plan.out.shape), dtype=torch.float32).pin_memory() for _ in range(2)]
    frames = [(h_feats, h_dist)] * K
    plan.run_frames(frames[:max(3, args.warmup)], [h_out[k & 1] for k in range(max(3, args.warmup))])
    torch.cuda.synchronize(dev)
    if world > 1:
        tdist.barrier()
    t0 = time.perf_counter()
    plan.run_frames(frames, [h_out[k & 1] for k in range(K)])
    e2e_tot = 1e3 * (time.perf_counter() - t0)
    per_rank_ms = [t / K for t in gather_scalars(tot_ms, dev)]
    multi = None
    if world > 1:
        # verification outside the timed region: every rank's map to rank 0,
        # which recomputes each sample in one process and compares the bits
        plan.run(feats, dist)
        full = gather_maps(plan.out.view(1, spec.channels, grid.nx, grid.ny).clone(), world)
        if rank == 0:
            same = []
            for r in range(world):
                (sd,) = sample_seeds(world, r, world)
                _, fr, lr, _ = bp.gen_workload(
                    bp.WorkloadSpec(spec.n_cameras, f, spec.grid, spec.channels, sd))
                ft = torch.from_numpy(fr).to(dev)[None]
                dt = bp.normalize_depth(torch.from_numpy(lr).to(dev))[None]
                want = plan.run(ft, dt).view(spec.channels, grid.nx, grid.ny)
                same.append(bool(torch.equal(full[r].to(dev), want)))
            multi = {"per_rank_step_ms": per_rank_ms,
                     "gathered_maps_bit_identical_to_single_process": all(same),
                     "collective_backend": tdist.get_backend()}
    tot_ms = max_over_ranks(tot_ms, dev)
    e2e_tot = max_over_ranks(e2e_tot, dev)

    variants = {}
    if rank == 0 and world == 1 and not args.no_variants:
        variants = run_variants(bp, torch, dev, spec, rig, feats, dist, cache, grid, flush)
    clk = clocks.stop()

    # ---- roofline: the pooling step (both kernels of the tiled path) ------
    # compulsory bytes of one pool_interval over the reference formulation
    # (SURVEY.md §8d, S): features + dist + ranks + interval table + map
    n_in, n_int = cache.n_in_range, cache.n_intervals
    C, NHW, NDHW = spec.channels, spec.n_cameras * f.height * f.width, P
    alg_bytes = 4 * NHW * C + 4 * NDHW + 4 * n_in + 8 * n_int + 4 * C * grid.n_cells
    step_avg_s = statistics.mean(step_ms) * 1e-3
    peak, peak_src = measured_peak()
    achieved = alg_bytes / step_avg_s / 1e9
    traffic = ncu_traffic(KERNEL_KEYS)
    # per kernel: the bytes each one moves (the segment rows go through L2)
    n_seg = plan._tile.n_seg
    n_groups_rec = n_in  # one 4-byte record per in-range point
    p1_bytes = 4 * NHW * C + 4 * NDHW + 4 * n_groups_rec + 4 * n_seg + 4 * C * n_seg
    p2_bytes = 4 * C * n_seg + 4 * (grid.n_cells + 1) + 4 * C * grid.n_cells
    p1_s, p2_s = statistics.mean(p1_ms) * 1e-3, statistics.mean(p2_ms) * 1e-3

    if rank != 0:
        if world > 1:
            tdist.destroy_process_group()
        return
    value = world * P * K / (tot_ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": max(3, args.warmup), "ms_per_step": tot_ms / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (reference gen_workload: PCG64 seed=rank, synthetic 6-camera rig)",
        "config": config_dict(spec),
        "parallelism": f"batch-sharded x{world} (1 sample/GPU, no collective in the step)",
        "timing": "CUDA events on the launching stream, L2 flushed (512 MiB write) before every step",
        "latency_ms": {"step_median": statistics.median(step_ms), "step_min": min(step_ms),
                       "tile_reduce_median": statistics.median(p1_ms),
                       "cell_combine_median": statistics.median(p2_ms),
                       "split_step_median": statistics.median(split_ms),
                       "step": "PoolPlan.run as one CUDA graph (tile_pool_kernel + "
                               "tile_finalize_kernel); per-kernel medians from the same two "
                               "launches as two graphs"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "pooling step = tile_pool_kernel + tile_finalize_kernel (the two "
                               "launches that replace interval_reduce), reference formulation",
                     "algorithmic_bytes_per_launch": alg_bytes, "peak_source": peak_src,
                     "frac_of_nominal_8TBs": achieved / 8000.0,
                     "kernels": {
                         "tile_pool_kernel": {"ms": statistics.mean(p1_ms), "bytes": p1_bytes,
                                              "GBps": p1_bytes / p1_s / 1e9,
                                              "frac": p1_bytes / p1_s / 1e9 / peak},
                         "tile_finalize_kernel": {"ms": statistics.mean(p2_ms), "bytes": p2_bytes,
                                                  "GBps": p2_bytes / p2_s / 1e9,
                                                  "frac": p2_bytes / p2_s / 1e9 / peak}}},
        "e2e": {"value": world * P * K / (e2e_tot * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": plan.h2d_bytes, "d2h_bytes_per_step": plan.d2h_bytes,
                "ms_per_step": e2e_tot / K,
                "path": "PoolPlan.run_frames: pinned H2D features+dist, pooling, D2H map per "
                        "frame; copies of consecutive frames overlap (wall clock)"},
        "gpu_launches": LAUNCHES_PER_STEP * K * world,
        "clocks": clk,
    }
    if multi is not None:
        line["multi_rank"] = multi
    if world == 1 and not args.no_cpu_baseline:
        times, threads, kind = time_cpu_reference(spec, args.cpu_seconds)
        v = P * len(times) / sum(times)
        line["cpu_baseline"] = {
            "value": v, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{len(times)} full nuScenes-shape pool_interval steps "
                      f"(median {1e3 * statistics.median(times):.1f} ms, ~{args.cpu_seconds:.0f} s "
                      f"of CPU), " + ("the reference itself (baseline/_ref, numba/OpenMP)"
                                      if kind == "reference" else "oracle C port, OpenMP")}
    if variants:
        line["variants"] = variants
    print(json.dumps(line), flush=True)
    if world > 1:
        tdist.destroy_process_group()


# ---------------------------------------------------------------------------
# configs B and H under the same launcher (batch-sharded, weak scaling)
# ---------------------------------------------------------------------------

def run_config_bh(args, bp, torch, tdist, dev, rank, world, local):
    """F: the fused lift+pool forward (bf16 logits and context -> fp32 map,
    the depth softmax formed per tile) through bp.pool_fused, one sample per
    GPU.  B: the training step -- tiled forward + tiled adjoint through the
    autograd op, batch 4 per GPU (samples rank*4 .. rank*4+3).  H: one
    high-res sample per GPU with the association rebuilt every step
    (CacheBuilder + PoolPlan.run_uncached).  Inputs resident in HBM, L2
    flushed before every step, CUDA events, max over ranks."""
    from paper_2205_13542_b200.shard import gather_scalars, max_over_ranks, sample_seeds

    name = args.config
    spec = bp.CONFIGS["H" if name == "H" else "S"]
    f = spec.frustum
    B_local = 4 if name == "B" else 1
    seeds = sample_seeds(world * B_local, rank, world)
    rig, _, _, grid = bp.gen_workload(spec)
    feats, dists, logits = [], [], []
    for sd in seeds:
        _, fr, lr, _ = bp.gen_workload(bp.WorkloadSpec(spec.n_cameras, f, spec.grid,
                                                       spec.channels, sd))
        feats.append(torch.from_numpy(fr))
        logits.append(torch.from_numpy(lr))
        dists.append(bp.normalize_depth(torch.from_numpy(lr).to(dev)).cpu())
    F = torch.stack(feats).to(dev)
    Dd = torch.stack(dists).to(dev)
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device=dev)
    if name == "F":
        cache = bp.build_cache(rig, f, grid, device=dev)
        LG = torch.stack(logits).to(dev).to(torch.bfloat16)
        CX = F.to(torch.bfloat16)

        def step():
            bp.pool_fused(LG, CX, cache, grid)
        launches = None
    elif name == "B":
        cache = bp.build_cache(rig, f, grid, device=dev)
        Fg = F.clone().requires_grad_(True)
        Dg = Dd.clone().requires_grad_(True)
        g = torch.randn((B_local, spec.channels, grid.nx, grid.ny), device=dev)

        def step():
            Fg.grad = None
            Dg.grad = None
            bp.bev_pool(Fg, Dg, cache, grid).backward(g)
        launches = None
    else:
        builder = bp.CacheBuilder(spec.n_cameras, f, grid, dev)
        cams = torch.from_numpy(bp.rig_rows(rig)).to(dev)
        plan = bp.PoolPlan(builder.build(cams), grid, spec.n_cameras, spec.channels, f.height,
                           f.width, f.depth_bins, 1, bp.Reducer.SUM, False, dev)

        def step():
            plan.run_uncached(builder, cams, F, Dd)
        launches = None
    stream = torch.cuda.current_stream(dev)
    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(max(3, args.warmup)):
        flush.zero_()
        step()
    K = args.steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize(dev)
    for k in range(K):
        flush.zero_()
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        tdist.barrier()
    step_ms = [e[0].elapsed_time(e[1]) for e in ev]
    clk = clocks.stop()
    per_rank = [t / K for t in gather_scalars(sum(step_ms), dev)]
    tot_ms = max_over_ranks(sum(step_ms), dev)
    if rank == 0:
        P = spec.n_points
        what = {"F": "fused bf16 lift+pool forward (bp.pool_fused: depth softmax per tile, "
                     "no dist or frustum tensor), 1 sample per GPU",
                "B": "training step: forward + tiled adjoint (autograd), batch 4 per GPU",
                "H": "high-res frame: association rebuilt every step + forward, 1 sample per GPU"
                }[name]
        cfg = config_dict(spec)
        cfg.update({"workload": f"config {name} ({what})", "batch_per_gpu": B_local})
        line = {"metric": METRIC, "value": world * B_local * P * K / (tot_ms * 1e-3),
                "unit": UNIT, "n_gpus": world, "steps": K, "warmup": max(3, args.warmup),
                "ms_per_step": tot_ms / K, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None,
                "dtype": "bf16 in / f32 accumulate" if name == "F" else "f32",
                "data": "synthetic (reference gen_workload)",
                "config": cfg,
                "parallelism": f"batch-sharded x{world}, no collective in the step",
                "timing": "CUDA events, L2 flushed (512 MiB write) before every step, max over ranks",
                "latency_ms": {"step_median": statistics.median(step_ms),
                               "per_rank_step_ms": per_rank},
                "e2e": None, "gpu_launches": launches, "clocks": clk}
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.destroy_process_group()


# ---------------------------------------------------------------------------
# other configurations (N=1): latency + roofline each, cold L2
# ---------------------------------------------------------------------------

def _timeit(torch, fn, flush, reps=10, warmup=3):
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        flush.zero_()
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def run_variants(bp, torch, dev, spec, rig, feats, dist, cache, grid, flush):
    peak, _ = measured_peak()
    f = spec.frustum
    C, P = spec.channels, spec.n_points
    NHW = spec.n_cameras * f.height * f.width
    n_in, n_int, n_cells = cache.n_in_range, cache.n_intervals, grid.n_cells
    out = {}

    def rec(name, ms, alg_bytes, **kw):
        gbs = alg_bytes / (ms * 1e-3) / 1e9
        out[name] = {"ms": ms, "points_per_s": P * kw.pop("samples", 1) / (ms * 1e-3),
                     "alg_bytes": alg_bytes, "GBps": gbs, "hbm_frac": gbs / peak, **kw}

    ref_bytes = 4 * NHW * C + 4 * P + 4 * n_in + 8 * n_int + 4 * C * n_cells
    for exact in (False, True):
        plan = bp.PoolPlan(cache, grid, spec.n_cameras, C, f.height, f.width, f.depth_bins, 1,
                           bp.Reducer.SUM, exact, dev)
        plan.transpose(feats)
        ms = _timeit(torch, lambda: plan.reduce(dist), flush)
        rec("interval_kernel_exact" if exact else "interval_kernel_fast", ms, ref_bytes)
        ms = _timeit(torch, lambda: plan.run(feats, dist), flush)
        rec("step_exact" if exact else "step_fast", ms, ref_bytes + 8 * NHW * C)
    for red in (bp.Reducer.MEAN, bp.Reducer.MAX):
        plan = bp.PoolPlan(cache, grid, spec.n_cameras, C, f.height, f.width, f.depth_bins, 1,
                           red, False, dev)
        ms = _timeit(torch, lambda: plan.run(feats, dist), flush)
        rec(f"step_fast_{red.value}", ms, ref_bytes + 8 * NHW * C)

    # materialised frustum: the paper's bev_pool input x (P, C)
    x = bp.lift_features(feats[0], dist[0])
    ms = _timeit(torch, lambda: bp.lift_features(feats[0], dist[0]), flush)
    rec("materialised_lift", ms, 4 * NHW * C + 4 * P + 4 * P * C)
    outx = torch.empty((C, n_cells), dtype=torch.float32, device=dev)
    from paper_2205_13542_b200 import _lib
    from paper_2205_13542_b200.bevgrid import ptr, stream_ptr
    from paper_2205_13542_b200.pooling import _scratch

    def pool_x():
        _lib.call("bvp_pool_lifted_f32", ptr(x), ptr(cache.d_ranks), ptr(cache.d_interval_starts),
                  ptr(cache.d_interval_cells), ptr(cache.d_cell_first), cache.schedule(), C,
                  grid.nx, grid.ny, 0,
                  ptr(outx), *_scratch(cache, 1, C, 0),
                  stream_ptr(dev))
    ms = _timeit(torch, pool_x, flush)
    rec("materialised_pool", ms, n_in * (4 * C + 4) + 8 * n_int + 4 * C * n_cells)
    del x

    # fused bf16 lift+pool: the tiled kernels with the depth softmax formed
    # per tile in shared memory (one CUDA graph, like the headline step)
    lg = torch.randn(dist.shape, device=dev).to(torch.bfloat16)
    cx = feats.to(torch.bfloat16)
    tp = cache.tile_plan(spec.n_cameras, f.height, f.width, f.depth_bins)
    fout = torch.empty((1, C, n_cells), dtype=torch.float32, device=dev)
    fused_fn = lambda: tp.pool_fused_bf16(lg, cx, 1, C, 0, fout)  # noqa: E731  (SUM)
    fused_fn()
    gf = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gf):
        fused_fn()
    ms = _timeit(torch, gf.replay, flush)
    rec("fused_bf16", ms, 2 * P + 2 * NHW * C + 4 * n_in + 8 * n_int + 4 * C * n_cells,
        path="tile_pool_kernel<bf16 fused> + tile_finalize_kernel (graph)")
    ms = _timeit(torch, lambda: bp.pool_fused(lg[0], cx[0], cache, grid), flush)
    rec("fused_bf16_api", ms, 2 * P + 2 * NHW * C + 4 * n_in + 8 * n_int + 4 * C * n_cells,
        path="bp.pool_fused (allocates its output every call)")

    # the reference's own calling convention: numpy in, numpy out, through
    # the drop-in pool_interval (pageable host arrays staged through pinned
    # buffers, the map copied back) -- wall clock per call, mean of 10
    import time
    fe_np = feats[0].cpu().numpy()
    di_np = dist[0].cpu().numpy()
    for _ in range(3):
        bp.pool_interval(fe_np, di_np, cache, grid)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(10):
        bp.pool_interval(fe_np, di_np, cache, grid)
    ms = 1e3 * (time.perf_counter() - t0) / 10
    rec("e2e_numpy_pool_interval", ms, ref_bytes,
        path="bp.pool_interval(numpy features, numpy dist) -> numpy map (the reference's "
             "convention; wall clock, pageable host arrays)")

    # cold association (geometry + sort + tables), no host sync
    builder = bp.CacheBuilder(spec.n_cameras, f, grid, dev)
    cams = torch.from_numpy(bp.rig_rows(rig)).to(dev)
    ms = _timeit(torch, lambda: builder.build(cams), flush)
    rec("association_cold", ms, 12 * P + 4 * n_in + 8 * n_cells + 8 * n_int)
    gbuilder = bp.CacheBuilder(spec.n_cameras, f, grid, dev, graph=True)
    ms = _timeit(torch, lambda: gbuilder.build(cams), flush)
    rec("association_cold_graph", ms, 12 * P + 4 * n_in + 8 * n_cells + 8 * n_int)
    ms = _timeit(torch, lambda: bp.reorder_weights(dist[0], cache), flush)
    rec("association_cached_reorder", ms, 4 * n_in + 4 * n_in + 4 * n_in)

    # paper's "before": prefix-sum pooling on the same GPU
    try:
        ms = _timeit(torch, lambda: bp.pool_prefixsum(feats[0], dist[0], cache, grid,
                                                      check_finite=False), flush, reps=3,
                     warmup=1)
        rec("prefixsum_baseline", ms, 8 * n_in * C * 3)
    except Exception as exc:  # pragma: no cover
        out["prefixsum_baseline"] = {"error": str(exc)}

    # training step, batch 4: tiled forward + tiled adjoint
    B = 4
    Fb = feats.expand(B, *feats.shape[1:]).contiguous().requires_grad_(True)
    Db = dist.expand(B, *dist.shape[1:]).contiguous().requires_grad_(True)
    g = torch.randn((B, C, grid.nx, grid.ny), device=dev)

    def train_step():
        o = bp.bev_pool(Fb, Db, cache, grid)
        o.backward(g)
    ms = _timeit(torch, train_step, flush)
    rec("training_b4_fwd_bwd", ms,
        B * (ref_bytes + 8 * NHW * C + 4 * C * n_cells + 4 * P + 4 * C * n_int + 4 * NHW * C
             + 4 * P), samples=B)
    # config F training step, batch 4: the fused forward and its tiled adjoint
    # (bf16 logits / context in, bf16 gradients out); bytes: forward and
    # backward each read the bf16 inputs, the map and its gradient, and the
    # backward writes both bf16 gradients
    LGb = lg.expand(B, *lg.shape[1:]).contiguous().requires_grad_(True)
    CXb = cx.expand(B, *cx.shape[1:]).contiguous().requires_grad_(True)

    def fused_train_step():
        LGb.grad = CXb.grad = None
        bp.bev_pool_fused(LGb, CXb, cache, grid).backward(g)
    ms = _timeit(torch, fused_train_step, flush)
    rec("training_fused_b4_fwd_bwd", ms,
        B * (3 * (2 * P + 2 * NHW * C) + 2 * 4 * C * n_cells + 8 * n_in), samples=B,
        path="bev_pool_fused forward + bvp_tile_fused_backward_bf16 (autograd)")

    # high-res stress: uncached geometry every frame + forward
    hs = bp.CONFIGS["H"]
    hrig, hf, hl, hgrid = bp.gen_workload(hs)
    hb = bp.CacheBuilder(hs.n_cameras, hs.frustum, hgrid, dev)
    hcams = torch.from_numpy(bp.rig_rows(hrig)).to(dev)
    hc = hb.build(hcams)
    hfe = torch.from_numpy(hf).to(dev)[None]
    hd = bp.normalize_depth(torch.from_numpy(hl).to(dev))[None]
    hplan = bp.PoolPlan(hc, hgrid, hs.n_cameras, hs.channels, hs.frustum.height, hs.frustum.width,
                        hs.frustum.depth_bins, 1, bp.Reducer.SUM, False, dev)

    def hframe():  # association beside the feature staging, then the pooling
        hplan.run_uncached(hb, hcams, hfe, hd)
    ms = _timeit(torch, hframe, flush)
    hP = hs.n_points
    hn_in, hn_int = hc.n_in_range, hc.n_intervals
    hbytes = (12 * hP + 4 * hn_in + 8 * hgrid.n_cells + 8 * hn_int) + (
        12 * hs.n_cameras * hs.frustum.height * hs.frustum.width * hs.channels + 4 * hP
        + 4 * hn_in + 8 * hn_int + 4 * hs.channels * hgrid.n_cells)
    out["highres_uncached_frame"] = {"ms": ms, "points_per_s": hP / (ms * 1e-3),
                                     "alg_bytes": hbytes, "GBps": hbytes / (ms * 1e-3) / 1e9,
                                     "hbm_frac": hbytes / (ms * 1e-3) / 1e9 / peak}
    # throughput of a frame stream: two builders / plans on two streams, so
    # frame k+1's association overlaps frame k's pooling (device time over
    # 20 frames, per frame)
    hb2 = bp.CacheBuilder(hs.n_cameras, hs.frustum, hgrid, dev)
    hplan2 = bp.PoolPlan(hb2.build(hcams), hgrid, hs.n_cameras, hs.channels, hs.frustum.height,
                         hs.frustum.width, hs.frustum.depth_bins, 1, bp.Reducer.SUM, False, dev)
    pipes = [(hb, hplan, torch.cuda.Stream(dev)), (hb2, hplan2, torch.cuda.Stream(dev))]
    n_frames = 20

    def hstream():
        cur = torch.cuda.current_stream(dev)
        for _, _, st in pipes:
            st.wait_stream(cur)
        for k in range(n_frames):
            b_, p_, st = pipes[k & 1]
            with torch.cuda.stream(st):
                p_.run_uncached(b_, hcams, hfe, hd)
        for _, _, st in pipes:
            cur.wait_stream(st)
    ms = _timeit(torch, hstream, flush) / n_frames
    out["highres_uncached_stream_per_frame"] = {
        "ms": ms, "points_per_s": hP / (ms * 1e-3), "alg_bytes": hbytes,
        "GBps": hbytes / (ms * 1e-3) / 1e9, "hbm_frac": hbytes / (ms * 1e-3) / 1e9 / peak,
        "note": "20 uncached frames, two builders on two streams (association of frame k+1 "
                "beside the pooling of frame k)"}
    return out


if __name__ == "__main__":
    main()
