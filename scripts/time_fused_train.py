"""Time config F training at S (batch B, default 4): the fused forward, the
tiled fused adjoint (bvp_tile_fused_backward_bf16) and the two-pass fallback
(bvp_fused_backward_bf16); cold L2, CUDA events, median of 20."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2205_13542_b200 as bp  # noqa: E402
from paper_2205_13542_b200 import _lib  # noqa: E402
from paper_2205_13542_b200.bevgrid import ptr, stream_ptr  # noqa: E402

spec = bp.CONFIGS["S"]
rig, feats_np, logits_np, grid = bp.gen_workload(spec)
cache = bp.build_cache(rig, spec.frustum, grid)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dev = torch.device("cuda")
lg = torch.from_numpy(logits_np).to(dev).to(torch.bfloat16).expand(B, *logits_np.shape).contiguous()
cx = torch.from_numpy(feats_np).to(dev).to(torch.bfloat16).expand(B, *feats_np.shape).contiguous()
N, D, H, W = logits_np.shape
C = feats_np.shape[1]
LG, CX = lg.clone().requires_grad_(True), cx.clone().requires_grad_(True)
g = torch.randn((B, C, grid.nx, grid.ny), device=dev)
gf = g.view(B, C, -1).contiguous()
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
tp = cache.tile_plan(N, H, W, D)
gl, gc = torch.empty_like(lg), torch.empty_like(cx)
ws = torch.empty(int(_lib.load().bvp_fused_backward_workspace_bytes(B, N, C, H, W, D,
                                                                    cache.n_int_max)),
                 dtype=torch.uint8, device=dev)


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
    LG.grad = CX.grad = None
    bp.bev_pool_fused(LG, CX, cache, grid).backward(g)


def tiled_bwd():
    tp.fused_backward_bf16(gf, lg, cx, B, C, _lib.BVP_SUM, gl, gc)


def gather_bwd():
    _lib.call("bvp_fused_backward_bf16", ptr(gf), ptr(lg), ptr(cx), ptr(cache.d_interval_starts),
              ptr(cache.d_interval_cells), ptr(cache.d_cell_first),
              ptr(cache.d_interval_of_point), B, N, C, H, W, D, grid.nx, grid.ny,
              cache.n_int_max, _lib.BVP_SUM, ptr(gl), ptr(gc), ptr(ws), ws.numel(),
              stream_ptr(dev))


print(f"config F training B={B}: fwd {t(lambda: bp.bev_pool_fused(lg, cx, cache, grid)):8.1f} us  "
      f"fwd+bwd {t(step):8.1f} us  tiled bwd {t(tiled_bwd):8.1f} us  "
      f"two-pass bwd {t(gather_bwd):8.1f} us")
