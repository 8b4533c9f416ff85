"""BEV pooling on the B200: the reference's pooling contract, GPU backends.

Drop-in for the reference's pooling module (pooling.py:1-261):

    value(g, c) = reducer over { dist[n,d,h,w] * features[n,c,h,w] :
                                 cell_of_point[(n,h,w,d)] = g },  empty -> 0

Backends (``pool(..., backend=...)``):
  interval   the fast path: cell-tiled interval reduction, one non-atomic
             store per (channel, cell) (csrc/pool_kernel.cuh).  ``exact=True``
             accumulates in 64 bits in rank order and is bit-identical to the
             reference's interval_reduce; ``exact=False`` accumulates in fp32.
  prefixsum  the paper's "before" (LSS cumsum trick), kept wasteful on purpose.
The reference's "naive" scatter is its CPU oracle; it is not a GPU backend.

Inputs may be numpy arrays (reference semantics: result is a numpy
BevFeatureMap; one H2D/D2H) or CUDA tensors (result stays on the device;
5-D (B, N, C, H, W) / (B, N, D, H, W) batches are accepted and pooled in one
launch into (B, C, nx, ny)).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .bevgrid import AssociationCache, BevGridSpec, cuda_device, ptr, stream_ptr, to_numpy
from .errors import ConfigurationError, StaleCacheError, UnsupportedReducerError, ValidationError
from .lift import nonfinite_flags

#: default accumulation: fp32 (fast; within 1.2e-7 of the reference at the
#: nuScenes shape, bar 1e-5).  exact=True reproduces the reference's 64-bit
#: interval_reduce bit for bit.
DEFAULT_EXACT = False


class Reducer(enum.Enum):
    SUM = "sum"
    MEAN = "mean"
    MAX = "max"

    @classmethod
    def parse(cls, name: str) -> "Reducer":
        try:
            return cls(name.lower())
        except ValueError:
            raise ConfigurationError(
                f"unknown reducer {name!r}; expected one of {[r.value for r in cls]}") from None


_MODE = {Reducer.SUM: _lib.BVP_SUM, Reducer.MEAN: _lib.BVP_MEAN, Reducer.MAX: _lib.BVP_MAX}


def _scratch(cache: AssociationCache, B: int, C: int, mode: int) -> tuple:
    """(pointer, bytes) of the fast kernels' scratch for this call shape."""
    t = cache.scratch(B, C, mode)
    return (None, 0) if t is None else (ptr(t), t.numel())

BACKENDS = ("naive", "prefixsum", "interval")

#: widest channel count of the tiled path (csrc/tile.cu: 4 x 32 lanes)
TILE_MAX_C = 128


def _tile_plan(cache: AssociationCache, N: int, H: int, W: int, D: int, C: int, mode: int,
               exact: int):
    """The pixel-column tiled reduction (csrc/tile.cu) pools SUM / MEAN in
    fast mode; MAX and exact mode use the interval kernels."""
    if exact or mode == _lib.BVP_MAX or C == 0 or C > TILE_MAX_C:
        return None
    return cache.tile_plan(N, H, W, D)


def _reducer(r) -> Reducer:
    return r if isinstance(r, Reducer) else Reducer.parse(str(r))


@dataclass(eq=False)
class BevFeatureMap:
    """Dense C x nx x ny float32 BEV features (numpy or CUDA tensor);
    batched CUDA results are B x C x nx x ny."""

    values: object
    grid: BevGridSpec

    def __post_init__(self):
        shape = tuple(self.values.shape)
        ok_rank = len(shape) == 3 or (len(shape) == 4 and isinstance(self.values, torch.Tensor))
        if not ok_rank or shape[-2:] != (self.grid.nx, self.grid.ny):
            raise ValidationError(
                f"values shape {shape} does not match grid ({self.grid.nx}, {self.grid.ny})")
        dt = self.values.dtype
        if dt not in (np.float32, torch.float32):
            raise ValidationError(f"values must be float32, got {dt}")

    @property
    def channels(self) -> int:
        return self.values.shape[-3]


# --------------------------------------------------------------------------
# input handling (reference _check_inputs, pooling.py:76-115)
# --------------------------------------------------------------------------

@dataclass
class _Inputs:
    feats: torch.Tensor     # (B, N, C, H, W) float32 CUDA, contiguous
    dist: torch.Tensor      # (B, N, D, H, W)
    host: bool
    batched: bool
    B: int
    N: int
    C: int
    H: int
    W: int
    D: int


def _check_inputs(features, dist, cache: AssociationCache, grid: BevGridSpec,
                  check_finite: bool = True) -> _Inputs:
    host = isinstance(features, np.ndarray)
    if host:
        if features.ndim != 4:
            raise ValidationError("features must be an (N, C, H, W) ndarray")
        if not isinstance(dist, np.ndarray) or dist.ndim != 4:
            raise ValidationError("dist must be an (N, D, H, W) ndarray")
        if features.dtype != np.float32 or dist.dtype != np.float32:
            raise ValidationError(
                f"features and dist must be float32, got {features.dtype} and {dist.dtype}")
    else:
        if not isinstance(features, torch.Tensor) or features.dim() not in (4, 5):
            raise ValidationError("features must be an (N, C, H, W) array or CUDA tensor")
        if not isinstance(dist, torch.Tensor) or dist.dim() != features.dim():
            raise ValidationError("dist must be an (N, D, H, W) tensor like features")
        if features.dtype != torch.float32 or dist.dtype != torch.float32:
            raise ValidationError(
                f"features and dist must be float32, got {features.dtype} and {dist.dtype}")
    batched = len(features.shape) == 5
    fs = tuple(features.shape) if batched else (1, *features.shape)
    ds = tuple(dist.shape) if batched else (1, *dist.shape)
    B, n, c, h, w = fs
    Bd, nd, d, hd, wd = ds
    if (B, n, h, w) != (Bd, nd, hd, wd):
        raise ValidationError(
            f"features {tuple(features.shape)} and dist {tuple(dist.shape)} disagree on (N, H, W)")
    dev = cuda_device(None if host else features.device)
    if host:
        ft = torch.from_numpy(np.ascontiguousarray(features)).to(dev).view(fs)
        dt = torch.from_numpy(np.ascontiguousarray(dist)).to(dev).view(ds)
    else:
        if not features.is_cuda or not dist.is_cuda:
            raise ValidationError("tensors must live on a CUDA device")
        ft = features.contiguous().view(fs)
        dt = dist.contiguous().view(ds)
    if check_finite:
        bad_f, bad_d = nonfinite_flags(ft, dt)  # one host sync for both
        if bad_f:
            raise ValidationError("features contain non-finite values")
        if bad_d:
            raise ValidationError("dist contains non-finite values")
    if cache.n_points != n * h * w * d:
        raise StaleCacheError(
            f"cache covers {cache.n_points} points but the workload has {n * h * w * d} "
            f"(N*H*W*D for N={n}, H={h}, W={w}, D={d})")
    if cache.grid is not None and cache.grid != grid:
        raise StaleCacheError("cache was built for a different BEV grid")
    if cache.frustum is not None and (
            cache.n_cameras != n or cache.frustum.height != h or cache.frustum.width != w
            or cache.frustum.depth_bins != d):
        raise StaleCacheError("cache was built for a different rig/frustum")
    if cache.grid is None and cache.n_intervals and int(cache.interval_cells.max()) >= grid.n_cells:
        raise StaleCacheError(
            "cache contains cell ids beyond this grid; it was built for a different grid")
    return _Inputs(ft, dt, host, batched, B, n, c, h, w, d)


def _finish(out: torch.Tensor, inp: _Inputs, grid: BevGridSpec) -> BevFeatureMap:
    shape = (inp.B, inp.C, grid.nx, grid.ny)
    v = out.view(shape)
    if not inp.batched:
        v = v[0]
    if inp.host:
        v = to_numpy(v)
    return BevFeatureMap(v, grid)


# --------------------------------------------------------------------------
# backends
# --------------------------------------------------------------------------

def pool_interval(features, dist, cache: AssociationCache, grid: BevGridSpec,
                  reducer=Reducer.SUM, *, exact: bool | None = None,
                  check_finite: bool = True) -> BevFeatureMap:
    """Interval-reduction pooling (reference pooling.py:206-221) on the GPU."""
    reducer = _reducer(reducer)
    inp = _check_inputs(features, dist, cache, grid, check_finite)
    cache = cache.for_grid(grid)
    out = torch.empty((inp.B, inp.C, grid.n_cells), dtype=torch.float32, device=inp.feats.device)
    exact = int(DEFAULT_EXACT if exact is None else exact)
    tp = _tile_plan(cache, inp.N, inp.H, inp.W, inp.D, inp.C, _MODE[reducer], exact)
    if tp is not None:
        tp.pool_f32(inp.feats, inp.dist, inp.B, inp.C, _MODE[reducer], out)
    elif inp.C:
        nhwc = torch.empty(inp.feats.numel(), dtype=torch.float32, device=inp.feats.device)
        _lib.call("bvp_pool_forward_f32", ptr(inp.feats), ptr(inp.dist), ptr(cache.d_ranks),
                  ptr(cache.d_interval_starts), ptr(cache.d_interval_cells),
                  ptr(cache.d_cell_first),
                  cache.schedule(inp.N, inp.H, inp.W, inp.D, exact=bool(exact)),
                  inp.B, inp.N, inp.C, inp.H, inp.W, inp.D,
                  grid.nx, grid.ny, cache.n_int_max, _MODE[reducer],
                  exact, ptr(out), ptr(nhwc), None,
                  *_scratch(cache, inp.B, inp.C, _MODE[reducer]), stream_ptr(inp.feats.device))
    return _finish(out, inp, grid)


def pool_prefixsum(features, dist, cache: AssociationCache, grid: BevGridSpec,
                   reducer=Reducer.SUM, *, check_finite: bool = True) -> BevFeatureMap:
    """The LSS cumsum baseline (reference pooling.py:162-196) on the GPU."""
    reducer = _reducer(reducer)
    if reducer is Reducer.MAX:
        raise UnsupportedReducerError(
            "prefix-sum cannot express max; use the interval backend")
    inp = _check_inputs(features, dist, cache, grid, check_finite)
    if inp.batched:
        raise ConfigurationError("the prefix-sum baseline pools one sample at a time")
    cache = cache.for_grid(grid)
    dev = inp.feats.device
    out = torch.empty((1, inp.C, grid.n_cells), dtype=torch.float32, device=dev)
    n_in, n_int = cache.n_in_range, cache.n_intervals
    ws = torch.empty(_lib.load().bvp_prefixsum_workspace_bytes(n_in, inp.C), dtype=torch.uint8,
                     device=dev)
    _lib.call("bvp_pool_prefixsum_f32", ptr(inp.feats), ptr(inp.dist), ptr(cache.d_ranks),
              ptr(cache.d_interval_starts), ptr(cache.d_interval_cells), n_in, n_int, inp.N,
              inp.C, inp.H, inp.W, inp.D, grid.n_cells, _MODE[reducer], ptr(out), ptr(ws),
              ws.numel(), stream_ptr(dev))
    return _finish(out, inp, grid)


def _fn_key(fn):
    """Stable cache key of a callable: bound methods by (object, name),
    functools.partials by their function and arguments, else the object."""
    import functools
    if isinstance(fn, functools.partial):
        return ("partial", _fn_key(fn.func), tuple(map(repr, fn.args)),
                tuple(sorted((k, repr(v)) for k, v in fn.keywords.items())))
    owner = getattr(fn, "__self__", None)
    if owner is not None:
        return ("method", id(owner), fn.__name__)
    return ("fn", fn)


class PoolPlan:
    """Pre-planned cached forward for fixed shapes (the serving loop).

    Output, NHWC staging and pinned host buffers are allocated once; ``run``
    is one C call on the current stream (features -> NHWC transpose beside the
    map's zero fill, then the interval reduction) with no validation and no
    host sync, so it can be captured in a CUDA graph.  ``run_host`` is the end-to-end
    drop-in for host (numpy) buffers: pinned H2D of features + dist, run,
    D2H of the (C, nx, ny) map.
    """

    def __init__(self, cache: AssociationCache, grid: BevGridSpec, n_cameras: int,
                 channels: int, height: int, width: int, depth_bins: int, batch: int = 1,
                 reducer=Reducer.SUM, exact: bool | None = None, device=None):
        self.dev = cuda_device(device if device is not None else cache.device)
        if cache.n_points != n_cameras * height * width * depth_bins:
            raise StaleCacheError("cache does not match the planned frustum")
        self.cache = cache.for_grid(grid)
        self.grid = grid
        self.B, self.N, self.C, self.H, self.W, self.D = (batch, n_cameras, channels, height,
                                                          width, depth_bins)
        self.mode = _MODE[_reducer(reducer)]
        self.exact = int(DEFAULT_EXACT if exact is None else exact)
        self._tile = _tile_plan(self.cache, n_cameras, height, width, depth_bins, channels,
                                self.mode, self.exact)
        f32 = dict(dtype=torch.float32, device=self.dev)
        self.out = torch.empty((batch, channels, grid.n_cells), **f32)
        self.nhwc = torch.empty(batch * n_cameras * height * width * channels, **f32)
        self._host = None
        self._scratch = _scratch(self.cache, batch, channels, self.mode)

    @property
    def feature_shape(self):
        return (self.B, self.N, self.C, self.H, self.W)

    @property
    def dist_shape(self):
        return (self.B, self.N, self.D, self.H, self.W)

    def transpose(self, features: torch.Tensor) -> None:
        _lib.call("bvp_to_nhwc_f32", ptr(features), self.B * self.N, self.C, self.H * self.W,
                  ptr(self.nhwc), stream_ptr(self.dev))

    @property
    def tiled(self) -> bool:
        """True when this plan pools through the pixel-column tiled path."""
        return self._tile is not None

    def phase(self, features: torch.Tensor, dist: torch.Tensor, which: int,
              out: torch.Tensor | None = None) -> torch.Tensor:
        """One launch of the tiled path alone (which = 1: the tile reduction
        into segment rows, 2: the per-cell combine into the map), for timing."""
        out = self.out if out is None else out
        flag = _lib.BVP_TILE_PHASE1 if which == 1 else _lib.BVP_TILE_PHASE2
        self._tile.pool_f32(features, dist, self.B, self.C, self.mode | flag, out)
        return out

    def prepare(self, features: torch.Tensor, zero: bool = True) -> None:
        """NHWC staging of the features beside the zero fill of the plan's
        output map (forked stream); follow with reduce(dist, zeroed=True).
        zero=False: the staging alone; reduce(dist) then zeroes the empty
        cells beside its kernels."""
        _lib.call("bvp_pool_prepare_f32", ptr(features), self.B, self.N, self.C, self.H, self.W,
                  ptr(self.nhwc), ptr(self.out) if zero else None, self.grid.n_cells,
                  stream_ptr(self.dev))

    def reduce(self, dist: torch.Tensor, out: torch.Tensor | None = None,
               zeroed: bool = False) -> torch.Tensor:
        """The interval reduction on the staged features.  zeroed=True: the
        plan's output was zero-filled by prepare() since it was last written
        (the reduction then skips its own zero fill)."""
        mode = self.mode | (_lib.BVP_OUT_ZEROED if zeroed and out is None else 0)
        out = self.out if out is None else out
        c = self.cache
        _lib.call("bvp_pool_forward_nhwc_f32", ptr(self.nhwc), ptr(dist), ptr(c.d_ranks),
                  ptr(c.d_interval_starts), ptr(c.d_interval_cells), ptr(c.d_cell_first),
                  c.schedule(self.N, self.H, self.W, self.D, exact=bool(self.exact)), self.B,
                  self.N, self.C, self.H, self.W, self.D, self.grid.nx, self.grid.ny, c.n_int_max,
                  mode, self.exact, ptr(out), None, *self._scratch, stream_ptr(self.dev))
        return out

    def run(self, features: torch.Tensor, dist: torch.Tensor,
            out: torch.Tensor | None = None) -> torch.Tensor:
        """features (B,N,C,H,W) / dist (B,N,D,H,W) contiguous float32 CUDA.
        One C call: the NHWC transpose and the map's zero fill run side by
        side (forked stream), then the interval reduction."""
        out = self.out if out is None else out
        if self._tile is not None:
            self._tile.pool_f32(features, dist, self.B, self.C, self.mode, out)
            return out
        c = self.cache
        _lib.call("bvp_pool_forward_f32", ptr(features), ptr(dist), ptr(c.d_ranks),
                  ptr(c.d_interval_starts), ptr(c.d_interval_cells), ptr(c.d_cell_first),
                  c.schedule(self.N, self.H, self.W, self.D, exact=bool(self.exact)), self.B,
                  self.N, self.C, self.H, self.W, self.D, self.grid.nx, self.grid.ny, c.n_int_max,
                  self.mode, self.exact, ptr(out), ptr(self.nhwc), None, *self._scratch,
                  stream_ptr(self.dev))
        return out

    def run_uncached(self, builder, cams: torch.Tensor, features: torch.Tensor,
                     dist: torch.Tensor) -> torch.Tensor:
        """One frame with the geometry rebuilt (config H): ``builder`` (the
        CacheBuilder whose buffers this plan's cache aliases) reassociates
        the rig ``cams`` while the features' staging and the map's zero fill
        run beside it on a side stream; then the reduction."""
        if self._tile is not None:
            # the builder rebuilds the tile plan this plan pools through
            self.cache = builder.build(cams).for_grid(self.grid)
            self._tile = _tile_plan(self.cache, self.N, self.H, self.W, self.D, self.C,
                                    self.mode, self.exact)
            return self.run(features, dist)
        cur = torch.cuda.current_stream(self.dev)
        side = self.__dict__.get("_side")
        if side is None:
            side = self._side = torch.cuda.Stream(self.dev)
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            self.prepare(features)
        # pool with the cache of THIS frame (its deferred units and exact
        # chunk list belong to it, not to the first frame's cache)
        self.cache = builder.build(cams).for_grid(self.grid)
        cur.wait_stream(side)
        return self.reduce(dist, zeroed=True)

    def graphed(self, fn, *tensors):
        """A CUDA graph of ``fn(*tensors)`` (the plan's launches on these
        buffers), captured once per buffer set and replayed after that: the
        frame loop then costs one host call instead of one per kernel."""
        key = (_fn_key(fn),) + tuple(t.data_ptr() for t in tensors)
        graphs = self.__dict__.setdefault("_graphs", {})
        g = graphs.get(key)
        if g is None:
            side = torch.cuda.Stream(self.dev)
            side.wait_stream(torch.cuda.current_stream(self.dev))
            with torch.cuda.stream(side):  # warm-up outside the capture
                fn(*tensors)
            torch.cuda.current_stream(self.dev).wait_stream(side)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn(*tensors)
            g.fn = fn  # keeps fn (and so its identity) alive with the graph
            graphs[key] = g
        return g

    def run_graphed(self, features: torch.Tensor, dist: torch.Tensor,
                    out: torch.Tensor | None = None) -> torch.Tensor:
        """``run`` replayed from a CUDA graph (same launches, same result)."""
        out = self.out if out is None else out
        self.graphed(self.run, features, dist, out).replay()
        return out

    def run_host(self, features, dist) -> np.ndarray:
        """Host buffers in, host BEV map out.  Pinned CPU tensors are copied
        straight to the device; numpy arrays are staged through pinned
        buffers first.  Returns a view of the pinned output buffer."""
        if self._host is None:
            pin = dict(dtype=torch.float32, pin_memory=True)
            self._host = (torch.empty(self.feature_shape, **pin), torch.empty(self.dist_shape, **pin),
                          torch.empty(tuple(self.out.shape), **pin),
                          torch.empty(self.feature_shape, dtype=torch.float32, device=self.dev),
                          torch.empty(self.dist_shape, dtype=torch.float32, device=self.dev))
        hf, hd, ho, df, dd = self._host
        if isinstance(features, torch.Tensor) and features.is_pinned():
            hf = features.view(self.feature_shape)
        else:
            hf.numpy()[...] = np.asarray(features, dtype=np.float32).reshape(self.feature_shape)
        if isinstance(dist, torch.Tensor) and dist.is_pinned():
            hd = dist.view(self.dist_shape)
        else:
            hd.numpy()[...] = np.asarray(dist, dtype=np.float32).reshape(self.dist_shape)
        df.copy_(hf, non_blocking=True)
        dd.copy_(hd, non_blocking=True)
        self.run(df, dd)
        ho.copy_(self.out, non_blocking=True)
        torch.cuda.current_stream(self.dev).synchronize()
        return ho.numpy().reshape(self.B, self.C, self.grid.nx, self.grid.ny)

    def run_frames(self, frames, outputs) -> None:
        """Serving loop over host frames: frames[k] = (features, dist) pinned
        CPU tensors of the planned shapes, outputs[k] a pinned CPU tensor of
        the map's shape.  Frame k's H2D (copy stream), pooling (current
        stream) and D2H (second copy stream) overlap frame k-1's D2H and
        frame k+1's H2D through two device buffer sets; returns when every
        output has landed."""
        cur = torch.cuda.current_stream(self.dev)
        if getattr(self, "_pipe", None) is None:
            f32 = dict(dtype=torch.float32, device=self.dev)
            self._pipe = dict(
                h2d=torch.cuda.Stream(self.dev), d2h=torch.cuda.Stream(self.dev),
                feats=[torch.empty(self.feature_shape, **f32) for _ in range(2)],
                dist=[torch.empty(self.dist_shape, **f32) for _ in range(2)],
                out=[torch.empty(tuple(self.out.shape), **f32) for _ in range(2)])
        pp = self._pipe
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        ev_free = [None, None]  # D2H of the buffer's previous frame done
        ev_used = [None, None]  # pooling of the buffer's previous frame done
        for k, ((hf, hd), ho) in enumerate(zip(frames, outputs)):
            i = k & 1
            with torch.cuda.stream(pp["h2d"]):
                if ev_used[i] is not None:
                    pp["h2d"].wait_event(ev_used[i])
                pp["feats"][i].copy_(hf.view(self.feature_shape), non_blocking=True)
                pp["dist"][i].copy_(hd.view(self.dist_shape), non_blocking=True)
                ev_in[i].record(pp["h2d"])
            cur.wait_event(ev_in[i])
            if ev_free[i] is not None:
                cur.wait_event(ev_free[i])
            self.run_graphed(pp["feats"][i], pp["dist"][i], pp["out"][i])
            ev_out[i].record(cur)
            ev_used[i] = torch.cuda.Event()
            ev_used[i].record(cur)
            with torch.cuda.stream(pp["d2h"]):
                pp["d2h"].wait_event(ev_out[i])
                ho.view(tuple(self.out.shape)).copy_(pp["out"][i], non_blocking=True)
                ev_free[i] = torch.cuda.Event()
                ev_free[i].record(pp["d2h"])
        pp["d2h"].synchronize()
        cur.synchronize()

    @property
    def h2d_bytes(self) -> int:
        return 4 * (int(np.prod(self.feature_shape)) + int(np.prod(self.dist_shape)))

    @property
    def d2h_bytes(self) -> int:
        return 4 * self.out.numel()


def pool_naive(features, dist, cache: AssociationCache, grid: BevGridSpec,
               reducer=Reducer.SUM, *, check_finite: bool = True) -> BevFeatureMap:
    """The reference's scatter backend (pooling.py:135-159) -- its results,
    on the GPU: every cell sums its points' fp64 products in original point
    order (which is rank order within a cell), MEAN divides by the count,
    MAX keeps the largest product.  Runs the exact-mode interval kernels;
    bit-identical to the reference's pool_naive."""
    reducer = _reducer(reducer)
    inp = _check_inputs(features, dist, cache, grid, check_finite)
    cache = cache.for_grid(grid)
    out = torch.empty((inp.B, inp.C, grid.n_cells), dtype=torch.float32, device=inp.feats.device)
    if inp.C:
        mode = _lib.BVP_MEAN_DIV if reducer is Reducer.MEAN else _MODE[reducer]
        nhwc = torch.empty(inp.feats.numel(), dtype=torch.float32, device=inp.feats.device)
        _lib.call("bvp_pool_forward_f32", ptr(inp.feats), ptr(inp.dist), ptr(cache.d_ranks),
                  ptr(cache.d_interval_starts), ptr(cache.d_interval_cells),
                  ptr(cache.d_cell_first),
                  cache.schedule(inp.N, inp.H, inp.W, inp.D, exact=True),
                  inp.B, inp.N, inp.C, inp.H, inp.W, inp.D,
                  grid.nx, grid.ny, cache.n_int_max, mode, 1, ptr(out), ptr(nhwc), None,
                  *_scratch(cache, inp.B, inp.C, _MODE[reducer]), stream_ptr(inp.feats.device))
    return _finish(out, inp, grid)


_BACKEND_FN = {"naive": pool_naive, "prefixsum": pool_prefixsum, "interval": pool_interval}

_PARALLELISM = [0]


def set_parallelism(n: int | None = None) -> int:
    """The reference sizes its CPU worker pool here (_threads.py:42-53).  The
    CUDA path has no host worker pool, so the count only records the
    request; it returns the count in effect like the reference (None reads
    BEVPOOL_THREADS, 0 = one per CPU)."""
    import os
    if n is None:
        raw = os.environ.get("BEVPOOL_THREADS", "0")
        try:
            n = int(raw)
        except ValueError:
            raise ConfigurationError(
                f"BEVPOOL_THREADS must be a non-negative integer, got {raw!r}") from None
        if n < 0:
            raise ConfigurationError(f"BEVPOOL_THREADS must be >= 0, got {n}")
    if n == 0:
        n = os.cpu_count() or 1
    _PARALLELISM[0] = max(1, int(n))
    return _PARALLELISM[0]


def get_parallelism() -> int:
    if not _PARALLELISM[0]:
        set_parallelism()
    return _PARALLELISM[0]


def pool(features, dist, cache, grid, reducer=Reducer.SUM, backend: str = "interval",
         **kwargs) -> BevFeatureMap:
    """Dispatch to the named backend (reference pooling.py:231-240)."""
    try:
        fn = _BACKEND_FN[backend]
    except KeyError:
        raise ConfigurationError(
            f"unknown backend {backend!r}; expected one of {BACKENDS}") from None
    return fn(features, dist, cache, grid, reducer, **kwargs)


def reorder_weights(dist, cache: AssociationCache):
    """Depth weights of the in-range points in cell-sorted order -- the cached
    association (reference pooling.py:243-261): a pure GPU gather by ranks."""
    host = isinstance(dist, np.ndarray)
    if len(dist.shape) != 4:
        raise ValidationError(f"dist must be (N, D, H, W), got {tuple(dist.shape)}")
    nd, d_, hd, wd = dist.shape
    if cache.n_points != nd * hd * wd * d_:
        raise StaleCacheError(
            f"cache covers {cache.n_points} points, dist implies {nd * hd * wd * d_}")
    dev = cache.device
    dt = (torch.from_numpy(np.ascontiguousarray(dist, dtype=np.float32)).to(dev) if host
          else dist.float().contiguous())
    n_in = cache.n_in_range
    w = torch.empty(n_in, dtype=torch.float32, device=dev)
    _lib.call("bvp_reorder_weights", ptr(dt), ptr(cache.d_ranks), n_in, nd, d_, hd, wd, ptr(w),
              stream_ptr(dev))
    return to_numpy(w) if host else w


# --------------------------------------------------------------------------
# the paper's materialised formulation and the fused bf16 path
# --------------------------------------------------------------------------

def lift_features(features: torch.Tensor, dist: torch.Tensor) -> torch.Tensor:
    """Materialise the frustum x (P, C) = dist (x) features in reference point
    order -- the input of the paper's bev_pool."""
    if features.dim() != 4 or dist.dim() != 4:
        raise ValidationError("features (N,C,H,W) and dist (N,D,H,W) expected")
    N, C, H, W = features.shape
    D = dist.shape[1]
    f = features.float().contiguous()
    d = dist.float().contiguous()
    x = torch.empty((N * H * W * D, C), dtype=torch.float32, device=f.device)
    _lib.call("bvp_lift_f32", ptr(f), ptr(d), N, C, H, W, D, ptr(x), stream_ptr(f.device))
    return x


def pool_lifted(x: torch.Tensor, cache: AssociationCache, grid: BevGridSpec,
                reducer=Reducer.SUM) -> BevFeatureMap:
    """Interval pooling of materialised frustum rows x (P, C) (fp32 accumulate)."""
    reducer = _reducer(reducer)
    if x.dim() != 2 or x.shape[0] != cache.n_points or x.dtype != torch.float32:
        raise ValidationError("x must be float32 (n_points, C)")
    cache = cache.for_grid(grid)
    C = x.shape[1]
    x = x.contiguous()
    out = torch.empty((C, grid.n_cells), dtype=torch.float32, device=x.device)
    _lib.call("bvp_pool_lifted_f32", ptr(x), ptr(cache.d_ranks), ptr(cache.d_interval_starts),
              ptr(cache.d_interval_cells), ptr(cache.d_cell_first),
              cache.schedule(), C,
              grid.nx, grid.ny,
              _MODE[reducer], ptr(out), *_scratch(cache, 1, C, _MODE[reducer]),
              stream_ptr(x.device))
    return BevFeatureMap(out.view(C, grid.nx, grid.ny), grid)


def pool_fused(logits: torch.Tensor, context: torch.Tensor, cache: AssociationCache,
               grid: BevGridSpec, reducer=Reducer.SUM) -> BevFeatureMap:
    """Fused lift+pool: pool(softmax_D(logits) (x) context) without forming
    either the depth distribution or the frustum; bf16 in, fp32 accumulate."""
    reducer = _reducer(reducer)
    if logits.dim() not in (4, 5) or context.dim() != logits.dim():
        raise ValidationError("logits (N,D,H,W) and context (N,C,H,W) expected")
    batched = logits.dim() == 5
    lg = (logits if batched else logits[None]).to(torch.bfloat16).contiguous()
    cx = (context if batched else context[None]).to(torch.bfloat16).contiguous()
    B, N, D, H, W = lg.shape
    C = cx.shape[2]
    if tuple(cx.shape) != (B, N, C, H, W):
        raise ValidationError("logits and context disagree on (B, N, H, W)")
    if cache.n_points != N * H * W * D:
        raise StaleCacheError("cache does not match the logits' frustum")
    cache = cache.for_grid(grid)
    dev = lg.device
    out = torch.empty((B, C, grid.n_cells), dtype=torch.float32, device=dev)
    tp = _tile_plan(cache, N, H, W, D, C, _MODE[reducer], 0)
    if tp is not None:  # softmax formed per tile in shared memory (csrc/tile.cu)
        tp.pool_fused_bf16(lg, cx, B, C, _MODE[reducer], out)
        v = out.view(B, C, grid.nx, grid.ny)
        return BevFeatureMap(v if batched else v[0], grid)
    ws = torch.empty(_lib.load().bvp_fused_workspace_bytes(B, N, C, H, W, D), dtype=torch.uint8,
                     device=dev)
    _lib.call("bvp_fused_pool_bf16", ptr(lg), ptr(cx), ptr(cache.d_ranks),
              ptr(cache.d_interval_starts), ptr(cache.d_interval_cells), ptr(cache.d_cell_first),
              cache.schedule(N, H, W, D),
              B, N, C, H, W, D, grid.nx, grid.ny, _MODE[reducer], ptr(out), ptr(ws), ws.numel(),
              *_scratch(cache, B, C, _MODE[reducer]), stream_ptr(dev))
    v = out.view(B, C, grid.nx, grid.ny)
    return BevFeatureMap(v if batched else v[0], grid)
