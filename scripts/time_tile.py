"""Time the pixel-column tiled path against the interval kernels (config S).

Cold L2 (512 MiB write before every rep), CUDA events on the current stream,
median of 20.  Prints one JSON line.
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_13542_b200 as bp  # noqa: E402


def timeit(fn, flush, reps=20, warm=3):
    st = torch.cuda.current_stream()
    for _ in range(warm):
        flush.zero_()
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


def main(name="S"):
    dev = torch.device("cuda")
    spec = bp.CONFIGS[name]
    f = spec.frustum
    rig, feats_np, logits_np, grid = bp.gen_workload(spec)
    cache = bp.build_cache(rig, f, grid)
    feats = torch.from_numpy(feats_np).to(dev)[None]
    dist = bp.normalize_depth(torch.from_numpy(logits_np).to(dev))[None]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    res = {"config": name}
    plan = bp.PoolPlan(cache, grid, spec.n_cameras, spec.channels, f.height, f.width,
                       f.depth_bins, 1, bp.Reducer.SUM, False, dev)
    res["tiled"] = plan.tiled
    tp = plan._tile
    res["n_seg"] = tp.n_seg
    res["max_seg"] = tp.max_seg
    g = plan.graphed(plan.run, feats, dist)
    res["step_graph_us"] = timeit(g.replay, flush)
    res["step_eager_us"] = timeit(lambda: plan.run(feats, dist), flush)
    res["phase1_us"] = timeit(lambda: plan.phase(feats, dist, 1), flush)
    plan.phase(feats, dist, 1)
    res["phase2_us"] = timeit(lambda: plan.phase(feats, dist, 2), flush)
    # the previous interval-kernel step on the same inputs
    old = bp.PoolPlan(cache, grid, spec.n_cameras, spec.channels, f.height, f.width,
                      f.depth_bins, 1, bp.Reducer.SUM, False, dev)
    old._tile = None
    go = old.graphed(old.run, feats, dist)
    res["interval_step_graph_us"] = timeit(go.replay, flush)
    a = plan.run(feats, dist).clone()
    b = old.run(feats, dist).clone()
    res["max_abs_diff_vs_interval"] = float((a - b).abs().max())
    # fused bf16
    lg = torch.from_numpy(logits_np).to(dev).to(torch.bfloat16)
    cx = torch.from_numpy(feats_np).to(dev).to(torch.bfloat16)
    res["fused_bf16_us"] = timeit(lambda: bp.pool_fused(lg, cx, cache, grid), flush)
    # per-frame association + plan (builder) and an uncached frame
    builder = bp.CacheBuilder(spec.n_cameras, f, grid, dev)
    cams = torch.from_numpy(bp.rig_rows(rig)).to(dev)
    res["builder_build_us"] = timeit(lambda: builder.build(cams), flush, reps=10)
    if builder.tplan is not None:
        res["tile_plan_build_us"] = timeit(lambda: builder.tplan.build(builder.bufs["cells"]),
                                           flush, reps=10)
    from paper_2205_13542_b200.bevgrid import TilePlan
    tp2 = TilePlan(spec.n_cameras, f.height, f.width, f.depth_bins, grid.n_cells, dev)
    res["tile_plan_build_sort_us"] = timeit(lambda: tp2.build(cache.d_cell_of_point), flush,
                                            reps=10)
    res["tile_plan_build_ranks_us"] = timeit(
        lambda: tp2.build(cache.d_cell_of_point, ranks=cache.d_ranks, counts=cache.d_counts),
        flush, reps=10)
    print(json.dumps(res))


if __name__ == "__main__":
    for n in (sys.argv[1:] or ["S"]):
        main(n)
