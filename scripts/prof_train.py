"""One config-B training step (batch 4 at S: forward + gather backward) after a
warm-up, for an ncu launch list:

    ncu --metrics gpu__time_duration.sum python scripts/prof_train.py
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
B = 4
feats = torch.from_numpy(fe).cuda()[None].expand(B, -1, -1, -1, -1).contiguous().requires_grad_(True)
dist = bp.normalize_depth(torch.from_numpy(lo).cuda())[None].expand(B, -1, -1, -1, -1).contiguous()
dist.requires_grad_(True)
g = torch.randn((B, spec.channels, grid.nx, grid.ny), device="cuda")
for _ in range(3):
    out = bp.bev_pool(feats, dist, cache, grid)
    out.backward(g)
torch.cuda.synchronize()
