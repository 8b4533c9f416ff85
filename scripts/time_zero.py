"""Where the map's zero fill goes (config S, bench timing: 512 MiB write flush
before every step, CUDA events, median of 40):
  A  staging graph [memset || NHWC transpose] | reduction graph   (bench today)
  B  staging graph [transpose] | reduction graph [zero-empty || chunk kernel]
  C  staging graph [zero-empty || transpose] | reduction graph
  A1, B1  the same launches as ONE graph (no split events).
  D1  one graph: zero-empty forked at the start, beside transpose + reduction.
  R   the reduction graph alone (map already zeroed; the roofline kernel)."""
import functools
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2205_13542_b200 as bp  # noqa: E402
from paper_2205_13542_b200 import _lib  # noqa: E402

spec = bp.CONFIGS["S"]
f = spec.frustum
rig, feats_np, logits_np, grid = bp.gen_workload(spec)
cache = bp.build_cache(rig, f, grid)
feats = torch.from_numpy(feats_np).cuda()[None]
dist = bp.normalize_depth(torch.from_numpy(logits_np).cuda())[None]
plan = bp.PoolPlan(cache, grid, 6, 80, f.height, f.width, f.depth_bins, 1, bp.Reducer.SUM)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
side = torch.cuda.Stream()


def stage_zero_empty(feats):
    cur = torch.cuda.current_stream()
    side.wait_stream(cur)
    with torch.cuda.stream(side):
        _lib.call("bvp_zero_empty_cells", cache.d_cell_first.data_ptr(), grid.n_cells, 80, 1,
                  plan.out.data_ptr(), side.cuda_stream)
    plan.prepare(feats, zero=False)
    cur.wait_stream(side)


def step_d():  # zero-empty forked at the step's start, beside transpose + reduction
    cur = torch.cuda.current_stream()
    side.wait_stream(cur)
    with torch.cuda.stream(side):
        _lib.call("bvp_zero_empty_cells", cache.d_cell_first.data_ptr(), grid.n_cells, 80, 1,
                  plan.out.data_ptr(), side.cuda_stream)
    plan.prepare(feats, zero=False)
    plan.reduce(dist, zeroed=True)
    cur.wait_stream(side)


def graph(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


variants = {
    "A": (graph(lambda: plan.prepare(feats)), graph(lambda: plan.reduce(dist, zeroed=True))),
    "B": (graph(lambda: plan.prepare(feats, zero=False)), graph(lambda: plan.reduce(dist))),
    "C": (graph(lambda: stage_zero_empty(feats)), graph(lambda: plan.reduce(dist, zeroed=True))),
    "A1": (graph(lambda: (plan.prepare(feats), plan.reduce(dist, zeroed=True))), None),
    "B1": (graph(lambda: (plan.prepare(feats, zero=False), plan.reduce(dist))), None),
    "D1": (graph(step_d), None),
    "R": (graph(lambda: plan.reduce(dist, zeroed=True)), None),
}
ref = plan.run(feats, dist).clone()
for name, (g1, g2) in variants.items():
    plan.out.fill_(float("nan"))
    g1.replay()
    if g2:
        g2.replay()
    torch.cuda.synchronize()
    same = bool(torch.equal(ref, plan.out))
    st, rd = [], []
    for i in range(43):
        flush.zero_()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        g1.replay()
        e[1].record()
        if g2:
            g2.replay()
        e[2].record()
        e[2].synchronize()
        if i >= 3:
            st.append(e[0].elapsed_time(e[1]) * 1e3)
            rd.append(e[1].elapsed_time(e[2]) * 1e3)
    tot = statistics.median([a + b for a, b in zip(st, rd)])
    print(f"{name:3s} first {statistics.median(st):6.1f} us  second {statistics.median(rd):6.1f} us"
          f"  step {tot:6.1f} us  same={same}")
