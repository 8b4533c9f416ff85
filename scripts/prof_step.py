"""The headline step as bench.py runs it (L2 flushed by a 512 MiB write, then
PoolPlan.run), repeated, for a precise per-kernel A/B under

    ncu --metrics gpu__time_duration.sum --cache-control none \
        -k "regex:tile_pool|tile_finalize" python scripts/prof_step.py [fused]

(--cache-control none keeps the flushed-L2 state the flush leaves, as in the
bench; the event clock on these boxes ticks in 2.048 us steps, too coarse for
a few-percent change).
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_13542_b200 as bp  # noqa: E402

spec = bp.CONFIGS["S"]
f = spec.frustum
rig, fe, lo, grid = bp.gen_workload(spec)
cache = bp.build_cache(rig, f, grid)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
if "fused" in sys.argv[1:]:
    lg = torch.from_numpy(lo).cuda().to(torch.bfloat16)
    cx = torch.from_numpy(fe).cuda().to(torch.bfloat16)
    step = lambda: bp.pool_fused(lg, cx, cache, grid)  # noqa: E731
else:
    feats = torch.from_numpy(fe).cuda()[None]
    dist = bp.normalize_depth(torch.from_numpy(lo).cuda())[None]
    plan = bp.PoolPlan(cache, grid, spec.n_cameras, spec.channels, f.height, f.width,
                       f.depth_bins)
    step = lambda: plan.run(feats, dist)  # noqa: E731
for _ in range(12):
    flush.zero_()
    step()
torch.cuda.synchronize()
