"""e2e serving loop (PoolPlan.run_frames) at the nuScenes shape, wall clock per
frame, with the staging forked (run) or serial (transpose + reduce)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2205_13542_b200 as bp  # noqa: E402

spec = bp.CONFIGS["S"]
f = spec.frustum
rig, feats_np, logits_np, grid = bp.gen_workload(spec)
cache = bp.build_cache(rig, f, grid)
dist = bp.normalize_depth(torch.from_numpy(logits_np).cuda())
h_feats = torch.from_numpy(feats_np).pin_memory()
h_dist = dist.cpu().pin_memory()
K = 60
for mode in ("forked", "serial", "forked", "serial"):
    plan = bp.PoolPlan(cache, grid, 6, 80, f.height, f.width, f.depth_bins, 1, bp.Reducer.SUM)
    if mode == "serial":
        def serial(fe, di, out=None, plan=plan):
            plan.transpose(fe)
            return plan.reduce(di, out)
        plan.run = serial
    h_out = [torch.empty(tuple(plan.out.shape)).pin_memory() for _ in range(2)]
    frames = [(h_feats, h_dist)] * K
    plan.run_frames(frames[:5], h_out * 3)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan.run_frames(frames, [h_out[k & 1] for k in range(K)])
    dt = (time.perf_counter() - t0) / K
    print(f"{mode:7s} {dt * 1e3:.3f} ms/frame")
