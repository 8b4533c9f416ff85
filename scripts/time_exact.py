"""Exact mode (and MAX) step times at config S, cold L2, CUDA events."""
import os, sys, statistics, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_13542_b200 as bp  # noqa: E402
spec = bp.CONFIGS["S"]; f = spec.frustum
rig, fe, lo, grid = bp.gen_workload(spec)
cache = bp.build_cache(rig, f, grid)
feats = torch.from_numpy(fe).cuda()[None]; dist = bp.normalize_depth(torch.from_numpy(lo).cuda())[None]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
res = {}
for name, red, exact in (("exact_sum", bp.Reducer.SUM, True), ("max", bp.Reducer.MAX, False),
                         ("exact_max", bp.Reducer.MAX, True), ("fast_sum", bp.Reducer.SUM, False)):
    plan = bp.PoolPlan(cache, grid, 6, 80, f.height, f.width, f.depth_bins, 1, red, exact)
    g = plan.graphed(plan.run, feats, dist)
    ts = []
    for i in range(23):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); b.synchronize()
        if i >= 3: ts.append(a.elapsed_time(b) * 1e3)
    res[name] = statistics.median(ts)
print(json.dumps(res))
