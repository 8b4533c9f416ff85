"""The tiled adjoint (bvp_tile_backward_f32; with the argument "fused" the
fused path's bvp_tile_fused_backward_bf16) at config S, batch 4, four
times, for an ncu launch list (compare with scripts/prof_train.py's gather
backward):

    ncu --metrics gpu__time_duration.sum -k regex:tile_ python scripts/prof_tile_bwd.py [fused]
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
B, C = 4, spec.channels
feats = torch.from_numpy(fe).cuda()[None].expand(B, -1, -1, -1, -1).contiguous()
dist = bp.normalize_depth(torch.from_numpy(lo).cuda())[None].expand(B, -1, -1, -1, -1).contiguous()
g = torch.randn((B, C, grid.n_cells), device="cuda")
tp = cache.tile_plan(spec.n_cameras, f.height, f.width, f.depth_bins)
gf, gw = torch.empty_like(feats), torch.empty_like(dist)
fused = len(sys.argv) > 1 and sys.argv[1] == "fused"
lg = torch.from_numpy(lo).cuda().to(torch.bfloat16)[None].expand(B, -1, -1, -1, -1).contiguous()
cx = feats.to(torch.bfloat16)
gl, gc = torch.empty_like(lg), torch.empty_like(cx)
for _ in range(4):
    if fused:
        tp.fused_backward_bf16(g, lg, cx, B, C, bp._lib.BVP_SUM, gl, gc)
    else:
        tp.backward_f32(g, feats, dist, B, C, bp._lib.BVP_SUM, gf, gw)
torch.cuda.synchronize()
