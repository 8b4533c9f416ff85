"""Time the unit kernel under different unit launch orders (BVP_UNIT_ORDER).

    python scripts/order_sweep.py "16,16,4" "8,8,1" ""
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2205_13542_b200 as bp  # noqa: E402

spec = bp.CONFIGS[os.environ.get("CFG", "S")]
f = spec.frustum
rig, feats_np, logits_np, grid = bp.gen_workload(spec)
cache = bp.build_cache(rig, f, grid)
feats = torch.from_numpy(feats_np).cuda()[None]
dist = bp.normalize_depth(torch.from_numpy(logits_np).cuda())[None]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
N, C = spec.n_cameras, spec.channels


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


ref = None
x = bp.lift_features(feats[0], dist[0])
for cfg in sys.argv[1:]:
    os.environ["BVP_UNIT_ORDER"] = cfg
    cache._host.pop("schedule", None)
    row = [f"order={cfg!r:12s}"]
    for exact in (False, True):
        plan = bp.PoolPlan(cache, grid, N, C, f.height, f.width, f.depth_bins, 1, bp.Reducer.SUM,
                           exact)
        plan.transpose(feats)
        out = plan.reduce(dist)
        if not exact:
            if ref is None:
                ref = out.clone()
            row.append(f"maxdiff {float((out - ref).abs().max()):.1e}")
        row.append(f"{'exact' if exact else 'fast'} {t(lambda: plan.reduce(dist)):7.1f} us")
    row.append(f"lifted {t(lambda: bp.pool_lifted(x, cache, grid)):7.1f} us")
    lg = torch.from_numpy(logits_np).cuda().bfloat16()
    cx = feats[0].bfloat16()
    row.append(f"fused {t(lambda: bp.pool_fused(lg, cx, cache, grid)):7.1f} us")
    print("  ".join(row), flush=True)
