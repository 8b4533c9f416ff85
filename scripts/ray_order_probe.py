"""Probe: reorder the cached chunk list so a warp's 8 lane groups walk cells
that share pixel columns (same camera ray), and time the interval kernel.

    python scripts/ray_order_probe.py
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
N, C, H, W, D = spec.n_cameras, spec.channels, f.height, f.width, f.depth_bins


def t(fn, n=30):
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


plan = bp.PoolPlan(cache, grid, N, C, H, W, D, 1, bp.Reducer.SUM, False)
plan.transpose(feats)
ref = plan.reduce(dist).clone()
nw = int(cache.d_work_counts[0])
work0 = cache.d_work[: 4 * nw].view(nw, 4).clone()
meta = cache.d_meta.view(-1, 2)
a = work0[:, 0].long()
ln = (work0[:, 1] - work0[:, 0]).long()
pix = meta[a, 0].long()
n_, hw = pix // (H * W), pix % (H * W)
h_, w_ = hw // W, hw % W
col = n_ * W + w_
bucket = cache.chunk - ln
ncol = N * W
variants = {
    "length, cell (current)": None,
    "length, column": bucket * ncol + col,
    "length, column, h0": (bucket * ncol + col) * H + h_,
    "column, length": col * (cache.chunk + 1) + bucket,
}
for name, key in variants.items():
    if key is None:
        w = work0
    else:
        order = torch.sort(key, stable=True).indices
        w = work0[order]
    cache.d_work[: 4 * nw].copy_(w.reshape(-1))
    out = plan.reduce(dist)
    md = float((out - ref).abs().max())
    print(f"{name:26s} kernel+combine {t(lambda: plan.reduce(dist)):7.1f} us  maxdiff {md:.1e}",
          flush=True)
cache.d_work[: 4 * nw].copy_(work0.reshape(-1))
