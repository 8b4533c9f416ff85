"""Drive the S-config kernels a few times for ncu (one GPU, no timing).

    ncu --set full -k regex:pool_tile_kernel -c 4 -o gpurun_out/prof python scripts/prof_pool.py
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2205_13542_b200 as bp  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
spec = bp.CONFIGS["S"]
f = spec.frustum
rig, feats_np, logits_np, grid = bp.gen_workload(spec)
cache = bp.build_cache(rig, f, grid)
feats = torch.from_numpy(feats_np).cuda()[None]
dist = bp.normalize_depth(torch.from_numpy(logits_np).cuda())[None]
for exact in ((False, True) if which == "all" else ((which == "exact"),)):
    plan = bp.PoolPlan(cache, grid, 6, 80, f.height, f.width, f.depth_bins, 1, bp.Reducer.SUM,
                       exact)
    for _ in range(reps):
        plan.run(feats, dist)
if which in ("all", "lifted"):
    x = bp.lift_features(feats[0], dist[0])
    for _ in range(reps):
        bp.pool_lifted(x, cache, grid)
if which in ("all", "fused"):
    for _ in range(reps):
        bp.pool_fused(torch.from_numpy(logits_np).cuda().bfloat16(), feats[0].bfloat16(), cache,
                      grid)
torch.cuda.synchronize()
print("done")
