"""Every CUDA path once at config T, for compute-sanitizer
(memcheck / racecheck / initcheck / synccheck):

    compute-sanitizer --tool racecheck python scripts/sanitize_T.py

fast (tiled) SUM / MEAN, MAX and exact (interval kernels), pool_naive,
the fused bf16 path and its tiled adjoint, the tiled adjoint (SUM / MEAN) and the gather backward
(MAX), a graph-captured PoolPlan step,
a per-frame CacheBuilder frame (association + tile plan), the reference-
shaped interval_reduce, the prefix-sum baseline, and the frustum / quantize
/ depth-check entry points.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_13542_b200 as bp  # noqa: E402

spec = bp.CONFIGS["T"]
f = spec.frustum
rig, feats_np, logits_np, grid = bp.gen_workload(spec)
dev = torch.device("cuda")
cache = bp.build_cache(rig, f, grid)
dist_np = bp.normalize_depth(logits_np)
for red in bp.Reducer:
    for exact in (False, True):
        bp.pool_interval(feats_np, dist_np, cache, grid, red, exact=exact)
    bp.pool_naive(feats_np, dist_np, cache, grid, red)
bp.pool_prefixsum(feats_np, dist_np, cache, grid)
feats = torch.from_numpy(feats_np).to(dev)
dist = torch.from_numpy(dist_np).to(dev)
lg = torch.from_numpy(logits_np).to(dev).to(torch.bfloat16)
bp.pool_fused(lg, feats.to(torch.bfloat16), cache, grid)
LG = lg[None].clone().requires_grad_(True)  # the fused path's tiled adjoint
CX = feats[None].to(torch.bfloat16).requires_grad_(True)
bp.bev_pool_fused(LG, CX, cache, grid).backward(
    torch.ones((1, spec.channels, grid.nx, grid.ny), device=dev))
F = feats[None].clone().requires_grad_(True)
D = dist[None].clone().requires_grad_(True)
for red in ("sum", "max"):  # tiled adjoint; gather backward
    F.grad = D.grad = None
    bp.bev_pool(F, D, cache, grid, red).backward(
        torch.ones((1, spec.channels, grid.nx, grid.ny), device=dev))
plan = bp.PoolPlan(cache, grid, spec.n_cameras, spec.channels, f.height, f.width, f.depth_bins)
plan.run_graphed(feats[None], dist[None])
builder = bp.CacheBuilder(spec.n_cameras, f, grid, tiles=True)
cams = torch.from_numpy(bp.rig_rows(rig)).to(dev)
uplan = bp.PoolPlan(builder.build(cams), grid, spec.n_cameras, spec.channels, f.height, f.width,
                    f.depth_bins)
uplan.run_uncached(builder, cams, feats[None], dist[None])
pts = bp.generate_frustum(rig, f)
bp.quantize_points(grid, pts)
bp.check_depth_distribution(dist)
from paper_2205_13542_b200 import _lib  # noqa: E402
from paper_2205_13542_b200.bevgrid import ptr, stream_ptr  # noqa: E402
out = torch.zeros((spec.channels, grid.n_cells), device=dev)
ft = feats.permute(0, 2, 3, 1).contiguous()
dt = dist.permute(0, 2, 3, 1).contiguous()
_lib.call("bvp_interval_reduce_f32", ptr(cache.d_ranks), ptr(cache.d_interval_starts),
          ptr(cache.d_interval_cells), cache.n_in_range, cache.n_intervals, ptr(dt), ptr(ft),
          ptr(out), grid.n_cells, f.height, f.width, f.depth_bins, spec.channels, 0,
          stream_ptr(dev))
torch.cuda.synchronize()
print("sanitize_T: all paths ran")
