"""Config H throughput: uncached frames back to back, one stream (latency
path, PoolPlan.run_uncached) vs two builders / plans alternating so frame
k+1's association overlaps frame k's pooling (two streams)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2205_13542_b200 as bp  # noqa: E402

spec = bp.CONFIGS["H"]
f = spec.frustum
rig, feats_np, logits_np, grid = bp.gen_workload(spec)
cams = torch.from_numpy(bp.rig_rows(rig)).cuda()
feats = torch.from_numpy(feats_np).cuda()[None]
dist = bp.normalize_depth(torch.from_numpy(logits_np).cuda())[None]
K = 40


def make():
    b = bp.CacheBuilder(spec.n_cameras, f, grid)
    p = bp.PoolPlan(b.build(cams), grid, spec.n_cameras, spec.channels, f.height, f.width,
                    f.depth_bins, 1, bp.Reducer.SUM)
    return b, p


b0, p0 = make()
b1, p1 = make()


def timed(fn):
    fn()
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    e.record()
    torch.cuda.synchronize()
    return a.elapsed_time(e) * 1e3 / K


def serial():
    for _ in range(K):
        p0.run_uncached(b0, cams, feats, dist)


streams = [torch.cuda.Stream(), torch.cuda.Stream()]


def pipelined():
    cur = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(cur)
    for k in range(K):
        s = streams[k & 1]
        b, p = (b0, p0) if k % 2 == 0 else (b1, p1)
        with torch.cuda.stream(s):
            p.run_uncached(b, cams, feats, dist)
    for s in streams:
        cur.wait_stream(s)


print(f"H uncached frames: serial {timed(serial):.1f} us/frame, "
      f"two streams {timed(pipelined):.1f} us/frame")
