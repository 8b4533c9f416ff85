"""Quick per-kernel timing at the S config (cold L2, CUDA events, median).

    python scripts/time_kernels.py [reps]
"""

import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2205_13542_b200 as bp  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
spec = bp.CONFIGS["S"]
f = spec.frustum
rig, feats_np, logits_np, grid = bp.gen_workload(spec)
cache = bp.build_cache(rig, f, grid)
feats = torch.from_numpy(feats_np).cuda()[None]
dist = bp.normalize_depth(torch.from_numpy(logits_np).cuda())[None]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def t(fn, n=reps):
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
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts), min(ts)


P, C = spec.n_points, spec.channels
NHW = 6 * f.height * f.width
alg = 4 * NHW * C + 4 * P + 4 * cache.n_in_range + 8 * cache.n_intervals + 4 * C * grid.n_cells
rows = []
for exact in (False, True):
    for red in (bp.Reducer.SUM, bp.Reducer.MAX):
        plan = bp.PoolPlan(cache, grid, 6, C, f.height, f.width, f.depth_bins, 1, red, exact)
        plan.transpose(feats)
        med, mn = t(lambda: plan.reduce(dist))
        rows.append((f"interval {'exact' if exact else 'fast '} {red.value}", med, mn, alg))
x = bp.lift_features(feats[0], dist[0])
med, mn = t(lambda: bp.pool_lifted(x, cache, grid))
rows.append(("materialised pool", med, mn, cache.n_in_range * (4 * C + 4) + 8 * cache.n_intervals
             + 4 * C * grid.n_cells))
del x
lg = torch.from_numpy(logits_np).cuda().bfloat16()
cx = feats[0].bfloat16()
med, mn = t(lambda: bp.pool_fused(lg, cx, cache, grid))
rows.append(("fused bf16 (3 kernels)", med, mn, 2 * P + 2 * NHW * C + 4 * NHW
             + 4 * cache.n_in_range + 8 * cache.n_intervals + 4 * C * grid.n_cells))
for name, med, mn, b in rows:
    print(f"{name:28s} median {med:8.1f} us  min {mn:8.1f} us  {b / med / 1e3:7.0f} GB/s "
          f"({b / med / 1e3 / 6538.6:.3f} of HBM)")
