"""Training: the interval pooling as a differentiable torch op (config B).

SUM / MEAN in fast mode run the pixel-column tiled reduction forward
(bvp_tile_pool_f32) and its adjoint backward (bvp_tile_backward_f32: the
same tiles and weight windows, every gradient row read once per segment);
MAX and exact mode run the cached interval reduction (bvp_pool_forward_f32)
and the atomic-free gather backward (bvp_pool_backward_f32,
csrc/backward.cu).  Both produce gradients for the context features and the
depth distribution.  MAX routes each output gradient to the first point
(rank order) attaining the max, recorded by the forward.  The reference has
no backward; tests/ check these against an fp64 restatement
that is itself checked against finite differences.
"""

from __future__ import annotations

import torch

from . import _lib
from .bevgrid import AssociationCache, BevGridSpec, ptr, stream_ptr
from .pooling import _MODE, BevFeatureMap, Reducer, _reducer, _scratch, _tile_plan


class _BevPoolFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, features, dist, cache: AssociationCache, nx: int, ny: int,
                reducer: Reducer, exact: bool):
        B, N, C, H, W = features.shape
        D = dist.shape[2]
        dev = features.device
        features = features.contiguous()
        dist = dist.contiguous()
        out = torch.empty((B, C, nx * ny), dtype=torch.float32, device=dev)
        tp = _tile_plan(cache, N, H, W, D, C, _MODE[reducer], int(exact))
        if tp is not None:  # the tiled path, forward and backward
            tp.pool_f32(features, dist, B, C, _MODE[reducer], out)
            ctx.cache, ctx.reducer, ctx.dims, ctx.tile = cache, reducer, (B, N, C, H, W, D, nx, ny), tp
            ctx.save_for_backward(features, dist)
            return out
        nhwc = torch.empty(features.numel(), dtype=torch.float32, device=dev)
        argmax = None
        if reducer is Reducer.MAX:
            argmax = torch.empty((B, cache.n_int_max, C), dtype=torch.int32, device=dev)
        _lib.call("bvp_pool_forward_f32", ptr(features), ptr(dist), ptr(cache.d_ranks),
                  ptr(cache.d_interval_starts), ptr(cache.d_interval_cells),
                  ptr(cache.d_cell_first),
                  cache.schedule(N, H, W, D, exact=bool(exact)),
                  B, N, C, H, W, D, nx, ny,
                  cache.n_int_max,
                  _MODE[reducer], int(exact), ptr(out), ptr(nhwc), ptr(argmax),
                  *_scratch(cache, B, C, _MODE[reducer]), stream_ptr(dev))
        ctx.cache, ctx.reducer, ctx.dims, ctx.tile = cache, reducer, (B, N, C, H, W, D, nx, ny), None
        ctx.save_for_backward(nhwc, dist, argmax)
        return out

    @staticmethod
    def backward(ctx, grad_out):
        cache, reducer = ctx.cache, ctx.reducer
        B, N, C, H, W, D, nx, ny = ctx.dims
        dev = grad_out.device
        g = grad_out.float().contiguous()
        need_f, need_w = ctx.needs_input_grad[0], ctx.needs_input_grad[1]
        gf = torch.empty((B, N, C, H, W), dtype=torch.float32, device=dev) if need_f else None
        gw = torch.empty((B, N, D, H, W), dtype=torch.float32, device=dev) if need_w else None
        if ctx.tile is not None:  # the tiled adjoint, on the forward's tiles
            features, dist = ctx.saved_tensors
            if need_f or need_w:
                ctx.tile.backward_f32(g, features, dist, B, C, _MODE[reducer], gf, gw)
            return gf, gw, None, None, None, None, None
        nhwc, dist, argmax = ctx.saved_tensors
        if need_f or need_w:
            ws = torch.empty(_lib.load().bvp_backward_workspace_bytes(B, C, cache.n_int_max),
                             dtype=torch.uint8, device=dev)
            _lib.call("bvp_pool_backward_f32", ptr(g), ptr(nhwc), ptr(dist),
                      ptr(cache.d_interval_starts), ptr(cache.d_interval_cells),
                      ptr(cache.d_cell_first), ptr(cache.d_interval_of_point), ptr(argmax), B, N,
                      C, H, W, D, nx, ny, cache.n_int_max, _MODE[reducer], ptr(gf), ptr(gw),
                      ptr(ws), ws.numel(), stream_ptr(dev))
        return gf, gw, None, None, None, None, None


def bev_pool(features: torch.Tensor, dist: torch.Tensor, cache: AssociationCache,
             grid: BevGridSpec, reducer=Reducer.SUM, exact: bool = False) -> torch.Tensor:
    """Differentiable pooling. features (N,C,H,W) or (B,N,C,H,W), dist
    (N,D,H,W) or (B,N,D,H,W), float32 CUDA -> (C,nx,ny) or (B,C,nx,ny)."""
    reducer = _reducer(reducer)
    batched = features.dim() == 5
    f = features if batched else features[None]
    d = dist if batched else dist[None]
    cache = cache.for_grid(grid)
    out = _BevPoolFn.apply(f.float(), d.float(), cache, grid.nx, grid.ny, reducer, exact)
    out = out.view(f.shape[0], f.shape[2], grid.nx, grid.ny)
    return out if batched else out[0]


def bev_pool_map(features, dist, cache, grid, reducer=Reducer.SUM) -> BevFeatureMap:
    return BevFeatureMap(bev_pool(features, dist, cache, grid, reducer), grid)


class _FusedPoolFn(torch.autograd.Function):
    """pool(softmax_D(logits) (x) context), bf16 in: the tiled fused forward
    (csrc/tile.cu, softmax in shared memory) and its tiled adjoint
    (bvp_tile_fused_backward_bf16, csrc/tile_backward.cu); MAX and C > 128
    take the interval forward and bvp_fused_backward_bf16."""

    @staticmethod
    def forward(ctx, logits, context, cache: AssociationCache, grid: BevGridSpec,
                reducer: Reducer):
        from .pooling import pool_fused
        out = pool_fused(logits, context, cache, grid, reducer).values
        ctx.cache, ctx.grid, ctx.reducer = cache, grid, reducer
        ctx.save_for_backward(logits, context)
        return out.view(logits.shape[0], context.shape[2], grid.n_cells)

    @staticmethod
    def backward(ctx, grad_out):
        logits, context = ctx.saved_tensors
        cache, grid = ctx.cache, ctx.grid
        B, N, D, H, W = logits.shape
        C = context.shape[2]
        dev = grad_out.device
        g = grad_out.float().contiguous()
        tp = _tile_plan(cache, N, H, W, D, C, _MODE[ctx.reducer], 0)
        if tp is not None:  # one pass per tile, bf16 gradients out
            need_l, need_c = ctx.needs_input_grad[0], ctx.needs_input_grad[1]
            gl = torch.empty_like(logits) if need_l else None
            gc = torch.empty_like(context) if need_c else None
            if need_l or need_c:
                tp.fused_backward_bf16(g, logits, context, B, C, _MODE[ctx.reducer], gl, gc)
            return gl, gc, None, None, None
        gl = torch.empty_like(logits)
        gc = torch.empty_like(context)
        ws = torch.empty(int(_lib.load().bvp_fused_backward_workspace_bytes(
            B, N, C, H, W, D, cache.n_int_max)), dtype=torch.uint8, device=dev)
        _lib.call("bvp_fused_backward_bf16", ptr(g), ptr(logits), ptr(context),
                  ptr(cache.d_interval_starts), ptr(cache.d_interval_cells),
                  ptr(cache.d_cell_first), ptr(cache.d_interval_of_point), B, N, C, H, W, D,
                  grid.nx, grid.ny, cache.n_int_max, _MODE[ctx.reducer], ptr(gl), ptr(gc),
                  ptr(ws), ws.numel(), stream_ptr(dev))
        return gl, gc, None, None, None


def bev_pool_fused(logits: torch.Tensor, context: torch.Tensor, cache: AssociationCache,
                   grid: BevGridSpec, reducer=Reducer.SUM) -> torch.Tensor:
    """Differentiable fused lift+pool (config F): logits (N,D,H,W) /
    (B,N,D,H,W) and context (N,C,H,W) / (B,N,C,H,W), bf16 CUDA -> fp32
    (C,nx,ny) / (B,C,nx,ny).  Gradients flow to both (bf16).  SUM / MEAN."""
    reducer = _reducer(reducer)
    if reducer is Reducer.MAX:
        from .errors import UnsupportedReducerError
        raise UnsupportedReducerError("the fused path is differentiable for SUM and MEAN")
    batched = logits.dim() == 5
    lg = (logits if batched else logits[None]).to(torch.bfloat16).contiguous()
    cx = (context if batched else context[None]).to(torch.bfloat16).contiguous()
    cache = cache.for_grid(grid)
    out = _FusedPoolFn.apply(lg, cx, cache, grid, reducer)
    out = out.view(lg.shape[0], cx.shape[2], grid.nx, grid.ny)
    return out if batched else out[0]
