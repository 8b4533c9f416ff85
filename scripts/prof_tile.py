"""The headline step's two kernels, as bench.py launches them (config S,
PoolPlan.run), for ncu --set full:

    ncu --set full -k "regex:tile_pool_kernel|tile_finalize_kernel" -s 2 -c 2 python scripts/prof_tile.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_13542_b200 as bp  # noqa: E402

spec = bp.CONFIGS["S"]
f = spec.frustum
rig, feats_np, logits_np, grid = bp.gen_workload(spec)
cache = bp.build_cache(rig, f, grid)
feats = torch.from_numpy(feats_np).cuda()[None]
dist = bp.normalize_depth(torch.from_numpy(logits_np).cuda())[None]
plan = bp.PoolPlan(cache, grid, spec.n_cameras, spec.channels, f.height, f.width, f.depth_bins)
for _ in range(3):
    plan.run(feats, dist)
torch.cuda.synchronize()
