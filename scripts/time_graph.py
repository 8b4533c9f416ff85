"""Step time of PoolPlan.run: eager launches vs one CUDA graph replay (cold L2)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2205_13542_b200 as bp  # noqa: E402

spec = bp.CONFIGS["S"]
f = spec.frustum
rig, feats_np, logits_np, grid = bp.gen_workload(spec)
cache = bp.build_cache(rig, f, grid)
feats = torch.from_numpy(feats_np).cuda()[None]
dist = bp.normalize_depth(torch.from_numpy(logits_np).cuda())[None]
plan = bp.PoolPlan(cache, grid, 6, 80, f.height, f.width, f.depth_bins, 1, bp.Reducer.SUM)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def t(fn, n=30, do_flush=True):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(n):
        if do_flush:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    plan.run(feats, dist)
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    plan.run(feats, dist)
eager = t(lambda: plan.run(feats, dist))
graph = t(lambda: g.replay())
warm_e = t(lambda: plan.run(feats, dist), do_flush=False)
warm_g = t(lambda: g.replay(), do_flush=False)
ref = plan.run(feats, dist).clone()
g.replay()
torch.cuda.synchronize()
print(f"eager {eager:.1f} us  graph {graph:.1f} us  (warm L2: eager {warm_e:.1f} graph {warm_g:.1f})"
      f"  same={bool(torch.equal(ref, plan.out))}")

# the bench's split: staging graph | reduction graph
gt = plan.graphed(plan.prepare, feats)
import functools  # noqa: E402
gr = plan.graphed(functools.partial(plan.reduce, zeroed=True), dist)
gtr = lambda: (gt.replay(), gr.replay())  # noqa: E731
print(f"staging graph {t(lambda: gt.replay()):.1f} us  reduction graph "
      f"{t(lambda: gr.replay()):.1f} us  both {t(gtr):.1f} us  "
      f"transpose only {t(lambda: plan.transpose(feats)):.1f} us")
