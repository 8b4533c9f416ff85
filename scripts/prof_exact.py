"""Exact-mode step at config S (PoolPlan.run, exact=True), three runs after a
warm-up, for an ncu launch list:

    ncu --metrics gpu__time_duration.sum python scripts/prof_exact.py
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
feats = torch.from_numpy(fe).cuda()[None]
dist = bp.normalize_depth(torch.from_numpy(lo).cuda())[None]
red = bp.Reducer.MAX if "max" in sys.argv[1:] else bp.Reducer.SUM
plan = bp.PoolPlan(cache, grid, 6, 80, f.height, f.width, f.depth_bins, 1, red, True)
for _ in range(4):
    plan.run(feats, dist)
torch.cuda.synchronize()
