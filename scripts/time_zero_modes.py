"""PoolPlan.run at config S, batch 1 and 4, eager and graph-replayed, with the
empty cells zeroed beside the reduction (BVP_ZERO_BESIDE=1) or the whole map
memset beside the transpose (=0).  Cold L2, CUDA events, median of 30.  Each
setting in a child process (the switch is read once per process)."""
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1:
    sys.path.insert(0, ROOT)
    import torch
    import paper_2205_13542_b200 as bp
    spec = bp.CONFIGS["S"]
    f = spec.frustum
    rig, feats_np, logits_np, grid = bp.gen_workload(spec)
    cache = bp.build_cache(rig, f, grid)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    res = []
    for B in (1, 4):
        feats = torch.from_numpy(feats_np).cuda()[None].expand(B, -1, -1, -1, -1).contiguous()
        dist = bp.normalize_depth(torch.from_numpy(logits_np).cuda())[None].expand(
            B, -1, -1, -1, -1).contiguous()
        plan = bp.PoolPlan(cache, grid, 6, 80, f.height, f.width, f.depth_bins, B, bp.Reducer.SUM)
        g = plan.graphed(plan.run, feats, dist)
        for label, fn in (("eager", lambda: plan.run(feats, dist)), ("graph", g.replay)):
            for _ in range(3):
                flush.zero_()
                fn()
            ts = []
            for _ in range(30):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            res.append(f"B={B} {label} {statistics.median(ts):6.1f} us")
    print(f"BVP_ZERO_BESIDE={os.environ['BVP_ZERO_BESIDE']}: " + "  ".join(res), flush=True)
else:
    for z in ("0", "1", "0", "1"):
        subprocess.run([sys.executable, __file__, "child"], env={**os.environ, "BVP_ZERO_BESIDE": z})
