"""Time phase-2 variants (scripts/fin_lab.cu) on the real config-S plan:
flush L2 -> phase 1 -> [event] variant [event], median of 30; each output
is compared with the product kernel's map.

    python scripts/fin_lab.py
"""
import ctypes
import json
import os
import statistics
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import paper_2205_13542_b200 as bp  # noqa: E402

SO = os.path.join(HERE, "_fin_lab.so")


def main():
    if not os.path.exists(SO):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-shared", "-Xcompiler", "-fPIC", "-o", SO,
                               os.path.join(HERE, "fin_lab.cu")])
    lab = ctypes.CDLL(SO)
    dev = torch.device("cuda")
    spec = bp.CONFIGS["S"]
    f = spec.frustum
    rig, feats_np, logits_np, grid = bp.gen_workload(spec)
    cache = bp.build_cache(rig, f, grid)
    feats = torch.from_numpy(feats_np).to(dev)[None]
    dist = bp.normalize_depth(torch.from_numpy(logits_np).to(dev))[None]
    plan = bp.PoolPlan(cache, grid, spec.n_cameras, spec.channels, f.height, f.width,
                       f.depth_bins, 1, bp.Reducer.SUM, False, dev)
    tp = plan._tile
    ref = plan.run(feats, dist).clone()
    rows = tp.rows(1, spec.channels)
    n_cells, C = grid.n_cells, spec.channels
    out = torch.empty(C * n_cells, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    res = {}

    def lab_call(v):
        rc = lab.fin_lab(v, ctypes.c_void_p(rows.data_ptr()),
                         ctypes.c_void_p(tp.st.cell_seg_first), n_cells, C,
                         ctypes.c_void_p(out.data_ptr()),
                         ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert rc == 0, rc

    def graph(fn):
        s2 = torch.cuda.Stream()
        s2.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s2):
            fn()
        torch.cuda.current_stream().wait_stream(s2)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        return g

    def timeit(g, reps=100):
        """flush, then the graph between events; mean (the event clock ticks
        in 2.048 us steps on this box, jitter makes the mean finer)."""
        ts = []
        for i in range(reps + 5):
            flush.zero_()
            lab.fin_lab_spin(ctypes.c_longlong(100000), ctypes.c_void_p(st.cuda_stream))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            g.replay()
            b.record(st)
            b.synchronize()
            if i >= 5:
                ts.append(a.elapsed_time(b) * 1e3)
        return round(statistics.fmean(ts), 2)

    t1 = timeit(graph(lambda: plan.phase(feats, dist, 1)))
    res["phase1"] = t1
    res["product_step"] = timeit(graph(lambda: plan.run(feats, dist)))
    only = os.environ.get("LAB_VARIANTS")
    variants = [int(x) for x in only.split(",")] if only else range(lab.fin_lab_count())
    for v in variants:
        out.fill_(float("nan"))
        plan.phase(feats, dist, 1)
        lab_call(v)
        ok = bool(torch.equal(out.view_as(ref), ref))
        t = timeit(graph(lambda v=v: (plan.phase(feats, dist, 1), lab_call(v))))
        res[f"v{v}"] = (t, round(t - t1, 2), ok)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
