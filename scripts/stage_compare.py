"""Per-stage comparison with the reference on the same box:
the reference's build_cache, normalize_depth, reorder_weights and
pool_interval timed on all host cores (baseline/_ref, fresh process,
OPENBLAS_NUM_THREADS=1), next to the GPU path's equivalents (CUDA events,
L2 flushed before every rep, median).

    python scripts/stage_compare.py > profiles/r01/stages.txt
"""
import json
import os
import platform
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

REF = r"""
import json, os, sys, time
sys.path.insert(0, os.environ["BVP_REF_DIR"])
import bevpool as ref
from bevpool.bevgrid import BevGridSpec
from bevpool.geometry import FrustumSpec
cfgs = {"S": (6, 32, 88, 118, 0.5, 80, 54.0, 0.3), "H": (6, 64, 176, 118, 0.5, 80, 54.0, 0.15)}
out = {"threads": ref.get_parallelism()}
for name, (n, h, w, d, step, c, e, r) in cfgs.items():
    spec = ref.WorkloadSpec(n, FrustumSpec(h, w, 1.0, step, d),
                            BevGridSpec(-e, e, -e, e, -10.0, 10.0, r), c, 0)
    rig, feats, logits, grid = ref.gen_workload(spec)
    def t(fn, reps):
        fn()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
        return statistics.median(ts)
    import statistics
    reps = 7 if name == "S" else 3
    res = {"build_cache": t(lambda: ref.build_cache(rig, spec.frustum, grid), reps)}
    cache = ref.build_cache(rig, spec.frustum, grid)
    res["normalize_depth"] = t(lambda: ref.normalize_depth(logits), reps)
    dist = ref.normalize_depth(logits)
    res["reorder_weights"] = t(lambda: ref.reorder_weights(dist, cache), reps)
    res["pool_interval"] = t(lambda: ref.pool_interval(feats, dist, cache, grid, ref.Reducer.SUM),
                             reps)
    out[name] = res
print(json.dumps(out))
"""


def reference_times():
    threads = len(os.sched_getaffinity(0))
    env = dict(os.environ, BVP_REF_DIR=os.path.join(ROOT, "baseline", "_ref"),
               OPENBLAS_NUM_THREADS="1", BEVPOOL_THREADS=str(threads),
               NUMBA_NUM_THREADS=str(threads), NUMBA_CACHE_DIR="/tmp/bvp_numba_cache")
    res = subprocess.run([sys.executable, "-c", REF], capture_output=True, text=True, env=env,
                         timeout=1800)
    if res.returncode != 0:
        raise SystemExit(f"reference failed: {res.stderr[-800:]}")
    return json.loads(res.stdout.strip().splitlines()[-1])


def gpu_times():
    import torch

    import paper_2205_13542_b200 as bp

    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def t(fn, n=20):
        for _ in range(3):
            flush.zero_()
            fn()
        ts = []
        for _ in range(n):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        return statistics.median(ts)

    out = {}
    for name in ("S", "H"):
        spec = bp.CONFIGS[name]
        f = spec.frustum
        rig, feats_np, logits_np, grid = bp.gen_workload(spec)
        builder = bp.CacheBuilder(spec.n_cameras, f, grid)
        cams = torch.from_numpy(bp.rig_rows(rig)).cuda()
        cache = bp.build_cache(rig, f, grid)
        logits = torch.from_numpy(logits_np).cuda()
        dist = bp.normalize_depth(logits)
        feats = torch.from_numpy(feats_np).cuda()[None]
        plan = bp.PoolPlan(cache, grid, spec.n_cameras, spec.channels, f.height, f.width,
                           f.depth_bins, 1, bp.Reducer.SUM)
        out[name] = {
            "build_cache": t(lambda: builder.build(cams)),
            "normalize_depth": t(lambda: bp.normalize_depth(logits)),
            "reorder_weights": t(lambda: bp.reorder_weights(dist, cache)),
            "pool_interval": t(lambda: plan.run(feats, dist[None])),
        }
    return out


def main():
    ref = reference_times()
    gpu = gpu_times()
    cpu = platform.processor() or platform.machine()
    try:
        with open("/proc/cpuinfo") as fh:
            cpu = next(l.split(":", 1)[1].strip() for l in fh if l.startswith("model name"))
    except (OSError, StopIteration):
        pass
    print(f"host: {cpu}; os.cpu_count()={os.cpu_count()}, "
          f"sched_getaffinity={len(os.sched_getaffinity(0))}, reference threads={ref['threads']}")
    print("GPU: one B200; per-frame association = CacheBuilder.build (geometry + sort + tables"
          " + chunk list + point table); pool_interval = PoolPlan.run (staging + reduction)")
    print(f"{'config':6s} {'stage':16s} {'reference (CPU)':>16s} {'B200':>12s} {'speed-up':>9s}")
    for name in ("S", "H"):
        for stage in ("build_cache", "normalize_depth", "reorder_weights", "pool_interval"):
            r, g = ref[name][stage], gpu[name][stage]
            print(f"{name:6s} {stage:16s} {r * 1e3:13.2f} ms {g * 1e6:9.1f} us {r / g:8.0f}x")


if __name__ == "__main__":
    main()
