"""Per-launch profile target: one uncached association + pool frame at a config
(ncu --metrics gpu__time_duration.sum ... python scripts/prof_assoc.py H)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2205_13542_b200 as bp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "H"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
spec = bp.CONFIGS[name]
f = spec.frustum
rig, feats_np, logits_np, grid = bp.gen_workload(spec)
builder = bp.CacheBuilder(spec.n_cameras, f, grid)
cams = torch.from_numpy(bp.rig_rows(rig)).cuda()
cache = builder.build(cams)
feats = torch.from_numpy(feats_np).cuda()[None]
dist = bp.normalize_depth(torch.from_numpy(logits_np).cuda())[None]
plan = bp.PoolPlan(cache, grid, spec.n_cameras, spec.channels, f.height, f.width,
                   f.depth_bins, 1, bp.Reducer.SUM)
torch.cuda.synchronize()
for _ in range(reps):
    builder.build(cams)
    plan.run(feats, dist)
torch.cuda.synchronize()
