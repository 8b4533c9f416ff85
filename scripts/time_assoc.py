"""Cold association (CacheBuilder.build) eager vs graph-replayed, configs S
and H: flush L2 (512 MiB write) before each rep, CUDA events, mean of 50."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_13542_b200 as bp  # noqa: E402


def timeit(fn, flush, reps=50):
    st = torch.cuda.current_stream()
    ts = []
    for i in range(reps + 5):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        if i >= 5:
            ts.append(a.elapsed_time(b) * 1e3)
    return round(statistics.fmean(ts), 1)


def main():
    dev = torch.device("cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    res = {}
    for name in sys.argv[1:] or ["S", "H"]:
        spec = bp.CONFIGS[name]
        rig, _, _, grid = bp.gen_workload(spec)
        cams = torch.from_numpy(bp.rig_rows(rig)).to(dev)
        for label, kw in (("eager", {}), ("graph", {"graph": True}),
                          ("graph_tiles", {"graph": True, "tiles": True})):
            b = bp.CacheBuilder(spec.n_cameras, spec.frustum, grid, dev, **kw)
            res[f"{name}_{label}_us"] = timeit(lambda: b.build(cams), flush)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
