"""BEV grid, the point -> cell association cache, and its wire format.

Mirrors the reference's bevgrid module (bevgrid.py:1-298): same grid
semantics (half-open cells, interior boundaries go up, ix-major flat ids,
z only gates membership), same AssociationCache contract (stable ranks,
interval_starts / interval_cells) and the same BVPC file format.  The
association itself is built on the GPU (csrc/geometry.cu): fp64 frustum ->
ego -> cell in the reference's exact rounding order, then a stable LSD radix
sort and interval tables, bit-identical to ``bevpool.build_cache``.

The cache lives in HBM: ``AssociationCache`` holds device tensors (uint32
values stored in torch.int32) plus two tables the GPU kernels need and the
reference does not have -- ``cell_first`` (index of the first interval of
every cell, so any run of cells maps to its interval range in O(1)) and
``interval_of_point`` (for the gather backward) -- and a sentinel
``interval_starts[n_int] = n_in`` so no kernel needs host-side counts.
The reference-typed numpy views (``cache.ranks`` ...) are host copies made
on first access.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import ConfigurationError, FileFormatError, StaleCacheError
from .geometry import CameraCalibration, FrustumSpec, rig_rows

#: Sentinel cell id of points outside the grid (also the wire encoding).
OUT_OF_RANGE = 0xFFFFFFFF
TILE_CELLS = _lib.TILE_CELLS

_CACHE_MAGIC = b"BVPC"
_CACHE_VERSION = 1


@dataclass(frozen=True)
class BevGridSpec:
    """Metric extents and cell size of the BEV grid (reference bevgrid.py:30-68)."""

    x_min: float
    x_max: float
    y_min: float
    y_max: float
    z_min: float
    z_max: float
    r: float

    def __post_init__(self):
        if self.r <= 0:
            raise ConfigurationError(f"cell size must be positive, got {self.r}")
        if self.z_min >= self.z_max:
            raise ConfigurationError(f"need z_min < z_max, got [{self.z_min}, {self.z_max})")
        for axis, lo, hi in (("x", self.x_min, self.x_max), ("y", self.y_min, self.y_max)):
            span = hi - lo
            n = span / self.r
            if span <= 0 or abs(n - round(n)) > 1e-9 or round(n) < 1:
                raise ConfigurationError(
                    f"{axis} extent [{lo}, {hi}) is not a positive integer multiple of r={self.r}")

    @property
    def nx(self) -> int:
        return round((self.x_max - self.x_min) / self.r)

    @property
    def ny(self) -> int:
        return round((self.y_max - self.y_min) / self.r)

    @property
    def n_cells(self) -> int:
        return self.nx * self.ny

    def as_array(self) -> np.ndarray:
        return np.array([self.x_min, self.x_max, self.y_min, self.y_max, self.z_min, self.z_max,
                         self.r], dtype=np.float64)


#: Benchmark default of the reference: 102.4 m square at r = 0.4 m.
DEFAULT_GRID = BevGridSpec(-51.2, 51.2, -51.2, 51.2, -10.0, 10.0, 0.4)


def quantize(spec: BevGridSpec, p) -> int:
    """Flat cell id of one ego point (scalar helper, bevgrid.py:71-82)."""
    x, y, z = float(p[0]), float(p[1]), float(p[2])
    ix = int(np.floor((x - spec.x_min) / spec.r))
    iy = int(np.floor((y - spec.y_min) / spec.r))
    if 0 <= ix < spec.nx and 0 <= iy < spec.ny and spec.z_min <= z < spec.z_max:
        return ix * spec.ny + iy
    return OUT_OF_RANGE


def cuda_device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.ExtensionMissingError("a CUDA device is required (no CPU fallback)")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    if device.type != "cuda":
        raise ConfigurationError(f"device must be a CUDA device, got {device}")
    return device


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def to_numpy(t: torch.Tensor) -> np.ndarray:
    """A device tensor as a new numpy array, copied through a pinned block of
    torch's caching host allocator: a pageable .cpu() of a fresh array pays a
    page fault per 4 KiB (19 ms for the 41.5 MB nuScenes map, against 0.7 ms
    this way).  The array keeps its block alive; freed blocks are reused."""
    if not t.is_cuda:
        return t.numpy()
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h.numpy()


def _u32(t: torch.Tensor) -> np.ndarray:
    return to_numpy(t).view(np.uint32)


#: chunk length of the fast kernels' work list (csrc/work.cu); 0 disables it
CHUNK = 64
#: chunk order: 0 = longest first (cell order within a length); > 0 = by 2D
#: tiles of WORK_TILE x WORK_TILE cells, longest first within a tile
WORK_TILE = 0
#: chunk length of the exact mode's own chunk list: its lane groups sum whole
#: intervals up to this length in fp64; longer ones are walked in order by a
#: CTA each (pool_exact_long_kernel), so fewer, longer chunks suit it
EXACT_CHUNK = 128


def work_bounds(n_points: int, n_int_max: int, chunk: int) -> tuple[int, int, int]:
    """Host upper bounds of the chunk schedule's counts without a host sync:
    chunks <= n_int + n_in / chunk; split intervals hold > chunk points each;
    their partial slots <= 2 n_in / chunk."""
    return (n_int_max + n_points // chunk + 1, n_points // (chunk + 1) + 1,
            2 * n_points // chunk + 1)


class TilePlan:
    """Device plan of the pixel-column tiled reduction (csrc/tile.cu): the
    in-range points of every camera column tile grouped by cell, built on the
    GPU from cell_of_point (no host round trip).  ``exact_count``: read the
    segment count back once (one sync) and size the segment-row scratch to
    it; otherwise the scratch is sized for the worst case (one segment per
    point), which per-frame rebuilds use."""

    def __init__(self, N: int, H: int, W: int, D: int, n_cells: int, device):
        lib = _lib.load()
        self.dims = (N, H, W, D)
        self.n_cells = n_cells
        self.device = device
        nbytes = int(lib.bvp_tile_plan_bytes(N, H, W, D, n_cells))
        if nbytes == 0:
            raise ConfigurationError(f"frustum {self.dims} not supported by the tile plan")
        self.buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        self.ws = torch.empty(int(lib.bvp_tile_plan_workspace_bytes(N, H, W, D, n_cells)),
                              dtype=torch.uint8, device=device)
        self.st = _lib.TilePlanStruct()
        self.bound = N * H * W * D
        _lib.call("bvp_tile_plan_init", ctypes.byref(self.st), N, H, W, D, n_cells,
                  ptr(self.buf), nbytes, self.bound)
        self._rows = {}

    @staticmethod
    def supported(N: int, H: int, W: int, D: int, n_cells: int) -> bool:
        return bool(_lib.load().bvp_tile_plan_supported(N, H, W, D, n_cells))

    def build(self, cell_of_point: torch.Tensor, exact_count: bool = False, ranks=None,
              counts=None) -> "TilePlan":
        """ranks / counts: the association's (device), whose stable sort by
        tile replaces the per-tile sort (same plan, faster)."""
        if ranks is not None:
            _lib.call("bvp_build_tile_plan_ranks", ptr(cell_of_point), ptr(ranks), ptr(counts),
                      ctypes.byref(self.st), ptr(self.ws), self.ws.numel(),
                      stream_ptr(self.device))
        else:
            _lib.call("bvp_build_tile_plan", ptr(cell_of_point), ctypes.byref(self.st),
                      ptr(self.ws), self.ws.numel(), stream_ptr(self.device))
        if exact_count:
            self.fit()
        return self

    @property
    def max_seg(self) -> int:
        return int(self.st.max_seg)

    @property
    def n_seg(self) -> int:
        """Segment count of the last build (one host sync)."""
        off = self.st.n_seg - self.buf.data_ptr()
        n = int(self.buf[off:off + 8].view(torch.int64).item())
        if n < 0:
            raise ConfigurationError("tile plan overflow (a tile's weight window is too large)")
        return n

    def fit(self) -> "TilePlan":
        """Shrink the segment-row scratch to the built plan (one sync)."""
        self.st.max_seg = max(1, self.n_seg)
        self._rows.clear()
        return self

    def rows(self, B: int, C: int) -> torch.Tensor:
        """Segment-row scratch for B samples of C channels (kept per shape)."""
        key = (B, C)
        t = self._rows.get(key)
        if t is None:
            t = torch.empty(B * self.max_seg * max(C, 1), dtype=torch.float32, device=self.device)
            self._rows[key] = t
        return t

    def pool_f32(self, features: torch.Tensor, dist: torch.Tensor, B: int, C: int, mode: int,
                 out: torch.Tensor) -> None:
        rows = self.rows(B, C)
        _lib.call("bvp_tile_pool_f32", ptr(features), ptr(dist), ctypes.byref(self.st), B, C,
                  mode, ptr(rows), 4 * rows.numel(), ptr(out), stream_ptr(self.device))

    def backward_f32(self, grad_out: torch.Tensor, features: torch.Tensor, dist: torch.Tensor,
                     B: int, C: int, mode: int, grad_features, grad_dist) -> None:
        """The adjoint of pool_f32 (SUM / MEAN): grad_features / grad_dist
        (either may be None) from grad_out (B, C, n_cells)."""
        rows = self.rows(B, C)
        _lib.call("bvp_tile_backward_f32", ptr(grad_out), ptr(features), ptr(dist),
                  ctypes.byref(self.st), B, C, mode, ptr(rows), 4 * rows.numel(),
                  ptr(grad_features), ptr(grad_dist), stream_ptr(self.device))

    def pool_fused_bf16(self, logits: torch.Tensor, context: torch.Tensor, B: int, C: int,
                        mode: int, out: torch.Tensor) -> None:
        rows = self.rows(B, C)
        _lib.call("bvp_tile_pool_fused_bf16", ptr(logits), ptr(context), ctypes.byref(self.st),
                  B, C, mode, ptr(rows), 4 * rows.numel(), ptr(out), stream_ptr(self.device))

    def fused_backward_bf16(self, grad_out: torch.Tensor, logits: torch.Tensor,
                            context: torch.Tensor, B: int, C: int, mode: int, grad_logits,
                            grad_context) -> None:
        """The adjoint of pool_fused_bf16 (SUM / MEAN): bf16 grad_logits /
        grad_context (either may be None) from grad_out (B, C, n_cells) f32."""
        rows = self.rows(B, C)
        _lib.call("bvp_tile_fused_backward_bf16", ptr(grad_out), ptr(logits), ptr(context),
                  ctypes.byref(self.st), B, C, mode, ptr(rows), 4 * rows.numel(),
                  ptr(grad_logits), ptr(grad_context), stream_ptr(self.device))


@dataclass(eq=False)
class AssociationCache:
    """Device-resident association of every frustum point with its BEV cell.

    ``ranks`` lists the in-range point ids sorted by cell (stable); interval
    i covers ranks[interval_starts[i] : interval_starts[i+1]] and all its
    points share cell interval_cells[i].  Immutable after build.  ``nx, ny``
    is the grid shape the cell tables were cut for.
    """

    d_cell_of_point: torch.Tensor          # (P,)
    d_ranks: torch.Tensor                  # (>= n_in,)
    d_interval_starts: torch.Tensor        # (>= n_int + 1,) with sentinel
    d_interval_cells: torch.Tensor         # (>= n_int,)
    d_cell_first: torch.Tensor             # (n_cells + 1,)
    d_interval_of_point: torch.Tensor      # (P,)
    d_counts: torch.Tensor                 # (2,) int64: n_in, n_int
    d_meta: torch.Tensor                   # (2 * P,) per sorted point: row, weight index
    fingerprint: int
    nx: int
    ny: int
    n_cameras: int | None = None
    frustum: FrustumSpec | None = field(default=None, repr=False)
    grid: BevGridSpec | None = field(default=None, repr=False)
    meta_dims: tuple | None = None         # (N, H, W, D) d_meta was derived for
    # chunk schedule of the fast kernels (csrc/work.cu); None when CHUNK == 0
    d_work: torch.Tensor | None = None     # (4 * max_work,) chunks, longest first
    d_splits: torch.Tensor | None = None   # (4 * max_splits,) intervals cut into chunks
    d_work_counts: torch.Tensor | None = None  # (3,) int64: n_work, n_splits, n_partials
    max_work: int = 0
    max_splits: int = 0
    max_partials: int = 0
    chunk: int = 0
    _host_counts: tuple | None = field(default=None, repr=False)
    _host: dict = field(default_factory=dict, repr=False)

    # ---- sizes ----------------------------------------------------------
    @property
    def device(self) -> torch.device:
        return self.d_cell_of_point.device

    @property
    def n_cells(self) -> int:
        return self.nx * self.ny

    @property
    def n_points(self) -> int:
        return int(self.d_cell_of_point.shape[0])

    def _counts(self):
        if self._host_counts is None:
            c = self.d_counts.cpu().tolist()
            self._host_counts = (int(c[0]), int(c[1]))
        return self._host_counts

    @property
    def n_in_range(self) -> int:
        return self._counts()[0]

    @property
    def n_intervals(self) -> int:
        return self._counts()[1]

    @property
    def n_int_max(self) -> int:
        """Capacity of the interval tables (no host sync)."""
        return int(self.d_interval_cells.shape[0])

    def fit_launch(self) -> None:
        """Shrink the launch bounds to the exact chunk counts (one host sync)."""
        if self.d_work_counts is not None:
            w = self.d_work_counts.cpu().tolist()
            self.max_work, self.max_splits, self.max_partials = int(w[0]), int(w[1]), int(w[2])
        for k in [k for k in self._host if isinstance(k, tuple) and k[0] == "schedules"]:
            self._host.pop(k)
        self._host.pop("scratch", None)

    def schedule(self, N: int | None = None, H: int = 1, W: int = 1, D: int = 1, *,
                 exact: bool = False):
        """The bvp_schedule the C ABI takes; the point gather table is
        (re)derived for an (N, H, W, D) frustum (N=None: the caller does not
        read it, e.g. the materialised path).  exact=True: the exact mode's
        own chunk list (EXACT_CHUNK), built on first use."""
        if N is not None and self.meta_dims != (N, H, W, D):
            _lib.call("bvp_point_meta", ptr(self.d_ranks), ptr(self.d_counts), N, H, W, D,
                      ptr(self.d_meta), stream_ptr(self.device))
            self.meta_dims = (N, H, W, D)
        xw = self.exact_work() if exact and self.d_work is not None else None
        key = ("schedules", xw is not None)
        s = self._host.get(key)
        if s is None:
            work = (None, None, None, 0, 0, 0, 0)
            if xw is not None:
                work = (ptr(xw["work"]), ptr(xw["splits"]), ptr(xw["counts"]), *xw["bounds"],
                        EXACT_CHUNK)
            elif self.d_work is not None:
                work = (ptr(self.d_work), ptr(self.d_splits), ptr(self.d_work_counts),
                        self.max_work, self.max_splits, self.max_partials, self.chunk)
            s = _lib.Schedule(ptr(self.d_meta), *work)
            self._host[key] = s
        return s

    def tile_plan(self, N: int, H: int, W: int, D: int) -> "TilePlan | None":
        """The tiled reduction's plan for an (N, H, W, D) frustum (built on
        first use, one sync to size its scratch); None when the frustum is
        outside the tiled path's limits."""
        key = ("tile", N, H, W, D)
        if key not in self._host:
            plan = None
            if TilePlan.supported(N, H, W, D, self.n_cells) and self.n_points == N * H * W * D:
                plan = TilePlan(N, H, W, D, self.n_cells, self.device).build(
                    self.d_cell_of_point, exact_count=True, ranks=self.d_ranks,
                    counts=self.d_counts)
            self._host[key] = plan
        return self._host[key]

    def exact_work(self) -> dict:
        """The exact mode's chunk list: intervals of <= EXACT_CHUNK points as
        single chunks, longest first (one build per cache, stream ordered)."""
        xw = self._host.get("exact_work")
        if xw is None:
            dev, i32 = self.device, dict(dtype=torch.int32, device=self.device)
            n_int_max, P = self.n_int_max, int(self.d_ranks.numel())
            mw, ms, mp = work_bounds(P, n_int_max, EXACT_CHUNK)
            xw = dict(work=torch.empty(4 * mw, **i32), splits=torch.empty(4 * ms, **i32),
                      counts=torch.zeros(3, dtype=torch.int64, device=dev), bounds=(mw, ms, mp))
            ws = torch.empty(int(_lib.load().bvp_work_workspace_bytes(
                n_int_max, P, EXACT_CHUNK, self.nx, self.ny, 0)), dtype=torch.uint8, device=dev)
            _lib.call("bvp_make_work", ptr(self.d_interval_starts), ptr(self.d_interval_cells),
                      ptr(self.d_counts), n_int_max, P, EXACT_CHUNK, self.nx, self.ny, 0,
                      ptr(xw["work"]), ptr(xw["splits"]), ptr(xw["counts"]), ptr(ws), ws.numel(),
                      stream_ptr(dev))
            xw["ws"] = ws  # kept until the build has run (stream ordered)
            self._host["exact_work"] = xw
        return xw

    def scratch(self, B: int, C: int, mode: int) -> torch.Tensor | None:
        """Scratch of the fast kernels (split-interval partials), kept per
        (B, C, mode) shape."""
        n = int(_lib.load().bvp_pool_scratch_bytes(self.schedule(), B, C, mode))
        if n == 0:
            return None
        key = (B, C, mode == 2)
        pool = self._host.setdefault("scratch", {})
        t = pool.get(key)
        if t is None or t.numel() < n:
            t = torch.zeros(n, dtype=torch.uint8, device=self.device)  # counters start at 0
            pool[key] = t
        return t

    # ---- reference-typed host views ------------------------------------
    def _view(self, name, tensor, n):
        if name not in self._host:
            arr = _u32(tensor[:n]).copy()
            arr.flags.writeable = False
            self._host[name] = arr
        return self._host[name]

    @property
    def cell_of_point(self) -> np.ndarray:
        return self._view("cell_of_point", self.d_cell_of_point, self.n_points)

    @property
    def ranks(self) -> np.ndarray:
        return self._view("ranks", self.d_ranks, self.n_in_range)

    @property
    def interval_starts(self) -> np.ndarray:
        return self._view("interval_starts", self.d_interval_starts, self.n_intervals)

    @property
    def interval_cells(self) -> np.ndarray:
        return self._view("interval_cells", self.d_interval_cells, self.n_intervals)

    @property
    def interval_of_point(self) -> np.ndarray:
        return self._view("interval_of_point", self.d_interval_of_point, self.n_points)

    def for_grid(self, grid: BevGridSpec) -> "AssociationCache":
        """This cache with cell tables / chunk list cut for ``grid``'s shape.
        Caches loaded from disk carry no grid (reference bevgrid.py:110-113);
        their tables are re-derived once per pooling grid shape."""
        if (grid.nx, grid.ny) == (self.nx, self.ny):
            return self
        key = ("grid", grid.nx, grid.ny)
        if key not in self._host:
            self._host[key] = cache_from_cells(self.cell_of_point, grid.nx, grid.ny,
                                               self.fingerprint, self.n_cameras, self.frustum,
                                               self.grid, self.device)
        return self._host[key]


def _alloc(P: int, nx: int, ny: int, dev) -> dict:
    i32 = dict(dtype=torch.int32, device=dev)
    lib = _lib.load()
    n_cells = nx * ny
    n_int_max = min(n_cells, P)
    ws = max(lib.bvp_sort_workspace_bytes(P, n_cells),
             lib.bvp_work_workspace_bytes(n_int_max, P, CHUNK, nx, ny, WORK_TILE)
             if CHUNK > 0 else 0)
    work = {}
    if CHUNK > 0:
        mw, ms, mp = work_bounds(P, n_int_max, CHUNK)
        work = dict(work=torch.empty(4 * mw, **i32), splits=torch.empty(4 * ms, **i32),
                    work_counts=torch.zeros(3, dtype=torch.int64, device=dev),
                    work_bounds=(mw, ms, mp), n_int_max=n_int_max)
    return dict(
        **work,
        cells=torch.empty(P, **i32), ranks=torch.empty(P, **i32),
        starts=torch.empty(n_cells + 1, **i32), icells=torch.empty(n_cells, **i32),
        cell_first=torch.empty(n_cells + 1, **i32), iop=torch.empty(P, **i32),
        counts=torch.zeros(2, dtype=torch.int64, device=dev),
        meta=torch.empty(2 * P, **i32),
        ws=torch.empty(ws, dtype=torch.uint8, device=dev),
    )


def _make_schedule(b: dict, nx: int, ny: int, dev, dims=None, work_tile: int = WORK_TILE,
                   work_done: bool = False) -> None:
    """The chunk schedule (work) of the interval kernels and the point gather
    table (stream ordered, no sync)."""
    if "work" in b and not work_done:
        _lib.call("bvp_make_work", ptr(b["starts"]), ptr(b["icells"]), ptr(b["counts"]),
                  b["n_int_max"], b["ranks"].numel(), CHUNK, nx, ny, work_tile, ptr(b["work"]),
                  ptr(b["splits"]), ptr(b["work_counts"]), ptr(b["ws"]), b["ws"].numel(),
                  stream_ptr(dev))
    if dims is not None and not work_done:
        N, H, W, D = dims
        _lib.call("bvp_point_meta", ptr(b["ranks"]), ptr(b["counts"]), N, H, W, D,
                  ptr(b["meta"]), stream_ptr(dev))


def _cache_of(b: dict, fingerprint, nx, ny, n_cameras, frustum, grid, dims=None):
    """A cache over the buffers b; launch bounds are the capacities until
    fit_launch() (no host sync needed to pool)."""
    cache = AssociationCache(b["cells"], b["ranks"], b["starts"], b["icells"], b["cell_first"],
                             b["iop"], b["counts"], b["meta"], fingerprint, nx, ny, n_cameras,
                             frustum, grid, dims)
    if "work" in b:
        cache.d_work, cache.d_splits, cache.d_work_counts = b["work"], b["splits"], b["work_counts"]
        cache.max_work, cache.max_splits, cache.max_partials = b["work_bounds"]
        cache.chunk = CHUNK
    return cache


class CacheBuilder:
    """Re-usable GPU association builder: buffers and workspace are allocated
    once for a (frustum, grid) shape and every ``build`` reruns geometry +
    sort + interval tables + chunk list on the current stream with no host
    round trip (config H: uncached geometry every frame).  The returned cache
    aliases the builder's buffers until the next ``build``."""

    def __init__(self, n_cameras: int, frustum: FrustumSpec, grid: BevGridSpec, device=None,
                 sort_work: bool = False, tiles: bool = False, graph: bool = False):
        self.dev = cuda_device(device)
        # graph: the build's launches are captured once into a CUDA graph
        # and replayed (one host call per frame instead of ~20 launches)
        self.use_graph = graph
        self._graph = None
        self._cams = None
        self.n_cameras, self.frustum, self.grid = n_cameras, frustum, grid
        self.P = n_cameras * frustum.points_per_camera
        self.bufs = _alloc(self.P, grid.nx, grid.ny, self.dev)
        # per-frame rebuilds keep the chunk list in cell order (the length
        # sort costs more than it saves once per frame) and build it beside
        # the rank sort (own workspace); cached builds sort it
        self.work_tile = WORK_TILE if sort_work else -1
        self._grid_arr = grid.as_array()
        self._one_call = not sort_work and CHUNK > 0
        self.dims = (n_cameras, frustum.height, frustum.width, frustum.depth_bins)
        # tiles: rebuild the tiled reduction's plan with every association
        # (otherwise a cache builds it on first tiled use, with one sync)
        self.tplan = (TilePlan(*self.dims, grid.n_cells, self.dev)
                      if tiles and TilePlan.supported(*self.dims, grid.n_cells) else None)
        if self._one_call:
            b = self.bufs
            n = int(_lib.load().bvp_work_workspace_bytes(b["n_int_max"], self.P, CHUNK, grid.nx,
                                                         grid.ny, -1))
            b["wws"] = torch.empty(n, dtype=torch.uint8, device=self.dev)

    def build(self, cams: torch.Tensor, fingerprint: int = 0) -> AssociationCache:
        """cams: (N, 16) float64 CUDA tensor (see geometry.rig_rows)."""
        f, g = self.frustum, self.grid
        if cams.dtype != torch.float64 or cams.shape != (self.n_cameras, 16) or not cams.is_cuda:
            raise ConfigurationError("cams must be a CUDA float64 (N, 16) tensor")
        dims = (self.n_cameras, f.height, f.width, f.depth_bins)
        if not self.use_graph:
            return self._launch(cams.contiguous(), fingerprint)
        if self._graph is None:
            self._cams = torch.empty_like(cams, memory_format=torch.contiguous_format)
            self._cams.copy_(cams)
            side = torch.cuda.Stream(self.dev)
            side.wait_stream(torch.cuda.current_stream(self.dev))
            with torch.cuda.stream(side):  # warm-up (lazy attributes) outside the capture
                self._launch(self._cams, fingerprint)
            torch.cuda.current_stream(self.dev).wait_stream(side)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                self._launch(self._cams, fingerprint)
            self._graph = graph
        self._cams.copy_(cams)
        self._graph.replay()
        cache = _cache_of(self.bufs, fingerprint, g.nx, g.ny, self.n_cameras, f, g, dims)
        cache._host[("tile", *self.dims)] = self.tplan
        return cache

    def _launch(self, cams: torch.Tensor, fingerprint: int) -> AssociationCache:
        b, f, g = self.bufs, self.frustum, self.grid
        dims = (self.n_cameras, f.height, f.width, f.depth_bins)
        if self._one_call:
            _lib.call("bvp_build_association", ptr(cams), *dims, f.depth_min, f.depth_step,
                      self._grid_arr.ctypes.data, g.nx, g.ny, ptr(b["cells"]), ptr(b["ranks"]),
                      ptr(b["starts"]), ptr(b["icells"]), ptr(b["cell_first"]), ptr(b["iop"]),
                      ptr(b["counts"]), CHUNK, ptr(b["work"]), ptr(b["splits"]),
                      ptr(b["work_counts"]), ptr(b["meta"]), ptr(b["ws"]), b["ws"].numel(),
                      ptr(b["wws"]), b["wws"].numel(), stream_ptr(self.dev))
            cache = _cache_of(b, fingerprint, g.nx, g.ny, self.n_cameras, f, g, dims)
            return self._with_tiles(cache)
        _lib.call("bvp_build_cache", ptr(cams), self.n_cameras, f.height, f.width, f.depth_bins,
                  f.depth_min, f.depth_step, self._grid_arr.ctypes.data, g.nx, g.ny,
                  ptr(b["cells"]), ptr(b["ranks"]), ptr(b["starts"]), ptr(b["icells"]),
                  ptr(b["cell_first"]), ptr(b["iop"]), ptr(b["counts"]), ptr(b["ws"]),
                  b["ws"].numel(), stream_ptr(self.dev))
        _make_schedule(b, g.nx, g.ny, self.dev, dims, work_tile=self.work_tile)
        cache = _cache_of(b, fingerprint, g.nx, g.ny, self.n_cameras, f, g, dims)
        return self._with_tiles(cache)

    def _with_tiles(self, cache: AssociationCache) -> AssociationCache:
        """Rebuild the tiled reduction's plan from this frame's cells (stream
        ordered, no sync; scratch sized for the worst case) and attach it."""
        if self.tplan is not None:
            self.tplan.build(self.bufs["cells"], ranks=self.bufs["ranks"],
                             counts=self.bufs["counts"])
            cache._host[("tile", *self.dims)] = self.tplan
        else:
            cache._host[("tile", *self.dims)] = None  # per-frame caches pool with the interval kernels
        return cache


def build_cache(rig: list[CameraCalibration], frustum_spec: FrustumSpec,
                grid_spec: BevGridSpec, device=None) -> AssociationCache:
    """Project the rig's frustum, quantise and sort by cell -- on the GPU.

    Drop-in for bevgrid.build_cache (reference bevgrid.py:183-203); the
    arrays are bit-identical to the reference's.
    """
    cams = rig_rows(rig)
    builder = CacheBuilder(len(rig), frustum_spec, grid_spec, device, sort_work=True)
    cams_d = torch.from_numpy(cams).to(builder.dev)
    cache = builder.build(cams_d, fingerprint_inputs(rig, frustum_spec, grid_spec))
    cache._counts()  # one sync: sizes known on the host from here on
    cache.fit_launch()
    cache._host.pop(("tile", *builder.dims), None)  # the tile plan is built on first use
    return cache


def cache_from_cells(cell_of_point, nx: int, ny: int, fingerprint: int = 0, n_cameras=None,
                     frustum=None, grid=None, device=None) -> AssociationCache:
    """Association cache from given cell ids (a loaded file, a synthetic test
    cache) for an nx x ny grid: GPU stable sort + interval tables
    (bevgrid.py:142-158) + the chunk list."""
    dev = cuda_device(device)
    cells = np.ascontiguousarray(cell_of_point, dtype=np.uint32)
    P = int(cells.shape[0])
    n_cells = nx * ny
    if P == 0:
        raise ConfigurationError("cache must cover at least one point")
    valid = cells[cells != OUT_OF_RANGE]
    if valid.size and int(valid.max()) >= n_cells:
        raise StaleCacheError("cache contains cell ids beyond this grid")
    b = _alloc(P, nx, ny, dev)
    b["cells"].copy_(torch.from_numpy(cells.view(np.int32).copy()))
    _lib.call("bvp_sort_intervals", ptr(b["cells"]), P, n_cells, ptr(b["ranks"]),
              ptr(b["starts"]), ptr(b["icells"]), ptr(b["cell_first"]), ptr(b["iop"]),
              ptr(b["counts"]), ptr(b["ws"]), b["ws"].numel(), stream_ptr(dev))
    dims = None
    if frustum is not None and n_cameras is not None:
        dims = (n_cameras, frustum.height, frustum.width, frustum.depth_bins)
    _make_schedule(b, nx, ny, dev, dims)
    cache = _cache_of(b, fingerprint, nx, ny, n_cameras, frustum, grid, dims)
    cache._counts()
    cache.fit_launch()
    return cache


def ranks_and_intervals(cells: np.ndarray, n_cells: int | None = None):
    """GPU restatement of bevgrid.ranks_and_intervals: (ranks, starts, cells)."""
    cells = np.ascontiguousarray(cells, dtype=np.uint32)
    if cells.size == 0:
        e = np.empty(0, dtype=np.uint32)
        return e, e.copy(), e.copy()
    if n_cells is None:
        valid = cells[cells != OUT_OF_RANGE]
        n_cells = int(valid.max()) + 1 if valid.size else 1
    c = cache_from_cells(cells, 1, n_cells)
    return c.ranks.copy(), c.interval_starts.copy(), c.interval_cells.copy()


def fingerprint_inputs(rig, frustum: FrustumSpec, grid: BevGridSpec) -> int:
    """blake2b-64 of the canonical bytes of rig + specs (bevgrid.py:161-180)."""
    buf = bytearray(struct.pack("<I", len(rig)))
    for cam in rig:
        buf += struct.pack("<i4d", cam.camera_id, cam.fx, cam.fy, cam.cx, cam.cy)
        buf += cam.rotation.astype("<f8").tobytes() + cam.translation.astype("<f8").tobytes()
    buf += struct.pack("<II2dI", frustum.height, frustum.width, frustum.depth_min,
                       frustum.depth_step, frustum.depth_bins)
    buf += struct.pack("<7d", grid.x_min, grid.x_max, grid.y_min, grid.y_max, grid.z_min,
                       grid.z_max, grid.r)
    return int.from_bytes(hashlib.blake2b(bytes(buf), digest_size=8).digest(), "little")


def validate_cache(cache: AssociationCache, rig, frustum_spec, grid_spec) -> bool:
    return cache.fingerprint == fingerprint_inputs(rig, frustum_spec, grid_spec)


# ---- BVPC wire format (bevgrid.py:216-292): host I/O, not accelerated ------
def serialize_cache(cache: AssociationCache) -> bytes:
    out = bytearray(_CACHE_MAGIC) + struct.pack("<HQ", _CACHE_VERSION, cache.fingerprint)
    for arr in (cache.cell_of_point, cache.ranks, cache.interval_starts, cache.interval_cells):
        out += struct.pack("<Q", arr.shape[0]) + arr.astype("<u4").tobytes()
    return bytes(out)


def deserialize_cache(data: bytes, n_cells: int | None = None, device=None) -> AssociationCache:
    """Decode a BVPC blob and rebuild the device tables from its cell ids.

    The file's ranks / intervals must equal the deterministic GPU re-sort of
    its cell_of_point (they do for every file the reference writes)."""
    pos = 0

    def take(n, what):
        nonlocal pos
        if pos + n > len(data):
            raise FileFormatError(f"truncated while reading {what}", offset=pos)
        chunk = data[pos:pos + n]
        pos += n
        return chunk

    magic = take(4, "magic")
    if magic != _CACHE_MAGIC:
        raise FileFormatError(f"bad magic {magic!r}, expected {_CACHE_MAGIC!r}", offset=0)
    (version,) = struct.unpack("<H", take(2, "version"))
    if version != _CACHE_VERSION:
        raise FileFormatError(f"unsupported cache version {version}", offset=4)
    (fingerprint,) = struct.unpack("<Q", take(8, "fingerprint"))
    arrays = []
    for what in ("cell_of_point", "ranks", "interval_starts", "interval_cells"):
        (count,) = struct.unpack("<Q", take(8, f"{what} length"))
        arrays.append(np.frombuffer(take(4 * count, what), dtype="<u4").copy())
    if pos != len(data):
        raise FileFormatError("trailing bytes after cache payload", offset=pos)
    cells, ranks, starts, icells = arrays
    if cells.size == 0:  # no frustum has zero points; the device tables need one
        raise FileFormatError("empty association (cell_of_point has no entries)", offset=14)
    if n_cells is None:
        n_cells = int(icells.max()) + 1 if icells.size else 1
    cache = cache_from_cells(cells, 1, n_cells, fingerprint, device=device)
    if not (np.array_equal(cache.ranks, ranks) and np.array_equal(cache.interval_starts, starts)
            and np.array_equal(cache.interval_cells, icells)):
        raise FileFormatError("ranks / intervals inconsistent with cell_of_point")
    return cache


def save_cache(path, cache: AssociationCache) -> None:
    with open(path, "wb") as fh:
        fh.write(serialize_cache(cache))


def load_cache(path, n_cells: int | None = None, device=None) -> AssociationCache:
    with open(path, "rb") as fh:
        return deserialize_cache(fh.read(), n_cells, device)
