"""Time config B (training, batch 4 at S): forward + gather backward, and the
backward alone (cold L2, CUDA events, median of 20)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2205_13542_b200 as bp  # noqa: E402

spec = bp.CONFIGS["S"]
rig, feats_np, logits_np, grid = bp.gen_workload(spec)
cache = bp.build_cache(rig, spec.frustum, grid)
feats = torch.from_numpy(feats_np).cuda()
dist = bp.normalize_depth(torch.from_numpy(logits_np).cuda())
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
F = feats.expand(B, *feats.shape).contiguous().requires_grad_(True)
D = dist.expand(B, *dist.shape).contiguous().requires_grad_(True)
g = torch.randn((B, spec.channels, grid.nx, grid.ny), device="cuda")
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


def step():
    o = bp.bev_pool(F, D, cache, grid)
    o.backward(g)


out = bp.bev_pool(F, D, cache, grid)
print(f"B={B} fwd {t(lambda: bp.bev_pool(F, D, cache, grid)):8.1f} us  "
      f"fwd+bwd {t(step):8.1f} us")
