import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2205_13542_b200 as bp
spec = bp.CONFIGS["S"]
rig, f, l, grid = bp.gen_workload(spec)
cache = bp.build_cache(rig, spec.frustum, grid)
lg = torch.from_numpy(l).cuda().to(torch.bfloat16)
cx = torch.from_numpy(f).cuda().to(torch.bfloat16)
for _ in range(3):
    bp.pool_fused(lg, cx, cache, grid)
torch.cuda.synchronize()
