"""How the L2 flush between steps bills the step: the bench's staging graph |
reduction graph split (config S) after (a) a 512 MiB write flush (the dirty
flush lines are written back during the step), (b) the same write followed by
a 256 MiB read (L2 left holding clean, unrelated lines), (c) no flush."""
import functools
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
clean = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
acc = torch.empty((), dtype=torch.float32, device="cuda")
gt = plan.graphed(plan.prepare, feats)
gr = plan.graphed(functools.partial(plan.reduce, zeroed=True), dist)
gt0 = plan.graphed(functools.partial(plan.prepare, zero=False), feats)
gr0 = plan.graphed(plan.reduce, dist)


def run(pre, n=40, pair=None):
    gt, gr = pair or (globals()["gt"], globals()["gr"])
    for _ in range(3):
        pre()
        gt.replay()
        gr.replay()
    st, rd = [], []
    for _ in range(n):
        pre()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        gt.replay()
        e[1].record()
        gr.replay()
        e[2].record()
        e[2].synchronize()
        st.append(e[0].elapsed_time(e[1]) * 1e3)
        rd.append(e[1].elapsed_time(e[2]) * 1e3)
    return statistics.median(st), statistics.median(rd), statistics.median([a + b for a, b in zip(st, rd)])


modes = {
    "write flush": lambda: flush.zero_(),
    "write flush + clean read": lambda: (flush.zero_(), acc.copy_(clean.sum())),
    "no flush": lambda: None,
}
for name, pre in modes.items():
    s, r, t = run(pre)
    print(f"{name:26s} staging {s:6.1f} us  reduction {r:6.1f} us  step {t:6.1f} us")
    s, r, t = run(pre, pair=(gt0, gr0))
    print(f"{name:26s} staging {s:6.1f} us  reduction {r:6.1f} us  step {t:6.1f} us"
          "  (empty cells zeroed beside the reduction)")
ref = plan.run(feats, dist).clone()
plan.out.fill_(float("nan"))
gt0.replay()
gr0.replay()
torch.cuda.synchronize()
print("concurrent zero bit-identical to the memset path:", bool(torch.equal(ref, plan.out)))
