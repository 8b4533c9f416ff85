"""Cold association (uncached geometry) and pooling at configs S and H: CUDA
events, cold L2, median of 20; plus a launch breakdown target for ncu."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2205_13542_b200 as bp  # noqa: E402

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def t(fn, n=20):
    for _ in range(3):
        flush.zero_()
        fn()
    ts = []
    for _ in range(n):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


for name in sys.argv[1:] or ["S", "H"]:
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
    tb = t(lambda: builder.build(cams))
    tp = t(lambda: plan.run(feats, dist))

    def frame():
        plan.run_uncached(builder, cams, feats, dist)
    print(f"{name}: association {tb:8.1f} us  pool step {tp:8.1f} us  frame {t(frame):8.1f} us")
