"""CPU oracle for the BEV-pooling hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module, and only as the checker
(or as the CPU arm that is timed beside the GPU).  The product package
``paper_2205_13542_b200`` never imports it; its CUDA path fails loudly
when the extension is missing instead of falling back here.

Two layers:

* ``liboracle.so`` (oracle/bevpool_oracle.c): the geometry, the stable
  counting sort and the 64-bit interval reduction, restated in C with
  OpenMP.  Bit-exact against the reference (pinned by the SHA-256 digests
  in tests/golden/, produced by importing the reference itself).
* numpy restatements of the small host-side pieces (rig, PCG64 inputs,
  depth softmax, scatter oracle, backward, bf16 fused path).

Each function cites the reference file:line it restates (paths relative to
the reference's pkg/src/bevpool/).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

OUT_OF_RANGE = 0xFFFFFFFF  # bevgrid.py:24

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with oracle/Makefile (gcc is in the image)."""
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH)
        < os.path.getmtime(os.path.join(_HERE, "bevpool_oracle.c"))
    ):
        subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i32, i64, f64 = ctypes.c_int, ctypes.c_int64, ctypes.c_double
        L.oracle_frustum_cells.argtypes = [P, i32, i32, i32, i32, f64, f64, P, i32, i32, P]
        L.oracle_frustum_cells.restype = None
        L.oracle_ranks_and_intervals.argtypes = [P, i64, i64, P, P, P, P]
        L.oracle_ranks_and_intervals.restype = i32
        L.oracle_interval_reduce.argtypes = [P, i64, P, P, i64, P, P, P, i64,
                                             i32, i32, i32, i32, i32]
        L.oracle_interval_reduce.restype = None
        L.oracle_pool_interval.argtypes = [P, P, P, i64, P, P, i64, P, i64,
                                           i32, i32, i32, i32, i32, i32, P]
        L.oracle_pool_interval.restype = None
        L.oracle_max_threads.argtypes = []
        L.oracle_max_threads.restype = i32
        L.oracle_set_threads.argtypes = [i32]
        L.oracle_set_threads.restype = None
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------
# configurations (SURVEY.md §8 header; BASELINE.json configs)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Config:
    name: str
    n_cameras: int
    height: int
    width: int
    depth_bins: int
    depth_min: float
    depth_step: float
    channels: int
    extent: float
    r: float
    z_min: float = -10.0
    z_max: float = 10.0

    @property
    def grid(self):
        return (-self.extent, self.extent, -self.extent, self.extent,
                self.z_min, self.z_max, self.r)

    @property
    def nx(self):
        return int(round(2 * self.extent / self.r))

    @property
    def ny(self):
        return self.nx

    @property
    def n_cells(self):
        return self.nx * self.ny

    @property
    def n_points(self):
        return self.n_cameras * self.height * self.width * self.depth_bins


CONFIGS = {
    "T": Config("T", 1, 16, 44, 59, 1.0, 1.0, 32, 51.2, 0.8),
    "S": Config("S", 6, 32, 88, 118, 1.0, 0.5, 80, 54.0, 0.3),
    "H": Config("H", 6, 64, 176, 118, 1.0, 0.5, 80, 54.0, 0.15),
}


# --------------------------------------------------------------------------
# workload (workload.py)
# --------------------------------------------------------------------------

def synthetic_rig(n_cameras: int, height: int, width: int) -> np.ndarray:
    """Restates workload.py:70-106.  Returns (N, 16) float64 rows
    fx, fy, cx, cy, R (row-major cam->ego), t."""
    focal = 0.8 * width
    rows = []
    for k in range(n_cameras):
        yaw = 2.0 * np.pi * k / n_cameras
        cos, sin = np.cos(yaw), np.sin(yaw)
        rot = np.column_stack([np.array([sin, -cos, 0.0]),
                               np.array([0.0, 0.0, -1.0]),
                               np.array([cos, sin, 0.0])])
        t = np.array([1.5 * cos, 1.5 * sin, 1.6])
        rows.append(np.concatenate([[focal, focal, width / 2.0, height / 2.0],
                                    rot.reshape(-1), t]))
    return np.ascontiguousarray(np.array(rows, dtype=np.float64))


def gen_inputs(n_cameras, channels, height, width, depth_bins, seed):
    """Restates workload.py:119-124: PCG64(seed); features U[-1,1) first,
    then logits U[-3,3), both float32."""
    rng = np.random.Generator(np.random.PCG64(seed))
    features = rng.uniform(-1.0, 1.0, size=(n_cameras, channels, height, width)).astype(np.float32)
    logits = rng.uniform(-3.0, 3.0, size=(n_cameras, depth_bins, height, width)).astype(np.float32)
    return features, logits


def normalize_depth(logits: np.ndarray) -> np.ndarray:
    """Restates lift.py:28-31: fp64 max-subtracted softmax over axis 1,
    stored float32."""
    shifted = logits.astype(np.float64) - logits.max(axis=1, keepdims=True)
    np.exp(shifted, out=shifted)
    shifted /= shifted.sum(axis=1, keepdims=True)
    return shifted.astype(np.float32)


# --------------------------------------------------------------------------
# geometry + association (geometry.py, bevgrid.py) -- via liboracle.so
# --------------------------------------------------------------------------

def frustum_cells(cams, height, width, depth_bins, depth_min, depth_step,
                  grid, nx, ny) -> np.ndarray:
    cams = np.ascontiguousarray(cams, dtype=np.float64).reshape(-1, 16)
    g = np.ascontiguousarray(grid, dtype=np.float64)
    n = cams.shape[0]
    out = np.empty(n * height * width * depth_bins, dtype=np.uint32)
    lib().oracle_frustum_cells(_p(cams), n, height, width, depth_bins,
                               float(depth_min), float(depth_step), _p(g),
                               nx, ny, _p(out))
    return out


def ranks_and_intervals(cells: np.ndarray, n_cells: int):
    """Restates bevgrid.py:142-158 (stable sort by cell, interval starts)."""
    cells = np.ascontiguousarray(cells, dtype=np.uint32)
    P = cells.shape[0]
    ranks = np.empty(P, dtype=np.uint32)
    starts = np.empty(min(P, n_cells) or 1, dtype=np.uint32)
    icells = np.empty_like(starts)
    counts = np.zeros(2, dtype=np.int64)
    rc = lib().oracle_ranks_and_intervals(_p(cells), P, n_cells, _p(ranks),
                                          _p(starts), _p(icells), _p(counts))
    if rc != 0:
        raise ValueError(f"oracle_ranks_and_intervals failed ({rc})")
    n_in, n_int = int(counts[0]), int(counts[1])
    return ranks[:n_in].copy(), starts[:n_int].copy(), icells[:n_int].copy()


def build_cache(cfg: Config, cams=None) -> dict:
    """Restates bevgrid.py:183-203 (minus the host-side fingerprint)."""
    if cams is None:
        cams = synthetic_rig(cfg.n_cameras, cfg.height, cfg.width)
    cells = frustum_cells(cams, cfg.height, cfg.width, cfg.depth_bins,
                          cfg.depth_min, cfg.depth_step, cfg.grid, cfg.nx, cfg.ny)
    ranks, starts, icells = ranks_and_intervals(cells, cfg.n_cells)
    return dict(cell_of_point=cells, ranks=ranks, interval_starts=starts,
                interval_cells=icells)


# --------------------------------------------------------------------------
# pooling (pooling.py, _kernels.py)
# --------------------------------------------------------------------------

MODE = {"sum": 0, "mean": 1, "max": 2}


def pool_interval(features, dist, ranks, starts, icells, n_cells, mode="sum"):
    """Restates pooling.py:206-221 + _kernels.py:22-63 (64-bit accumulate in
    rank order).  Returns (C, n_cells) float32."""
    features = np.ascontiguousarray(features, dtype=np.float32)
    dist = np.ascontiguousarray(dist, dtype=np.float32)
    N, C, H, W = features.shape
    D = dist.shape[1]
    ranks = np.ascontiguousarray(ranks, dtype=np.uint32)
    starts = np.ascontiguousarray(starts, dtype=np.uint32)
    icells = np.ascontiguousarray(icells, dtype=np.uint32)
    out = np.empty((C, n_cells), dtype=np.float32)
    scratch = np.empty(max(1, N * H * W * (C + D)), dtype=np.float32)
    lib().oracle_pool_interval(_p(features), _p(dist), _p(ranks), ranks.size,
                               _p(starts), _p(icells), starts.size, _p(out),
                               n_cells, N, C, H, W, D, MODE[mode], _p(scratch))
    return out


def pool_naive(features, dist, cell_of_point, n_cells, mode="sum"):
    """Restates pooling.py:135-159: scatter in original point order, fp64
    bincount per channel (MAX: maximum.at, -inf -> 0)."""
    N, C, H, W = features.shape
    D = dist.shape[1]
    idx = np.nonzero(cell_of_point != OUT_OF_RANGE)[0].astype(np.int64)
    out = np.zeros((C, n_cells), dtype=np.float32)
    if idx.size == 0 or C == 0:
        return out
    cells = cell_of_point[idx].astype(np.int64)
    d = idx % D
    rest = idx // D
    w = rest % W
    rest //= W
    h = rest % H
    n = rest // H
    weights = dist[n, d, h, w].astype(np.float64)
    if mode == "max":
        for c in range(C):
            best = np.full(n_cells, -np.inf)
            np.maximum.at(best, cells, weights * features[n, c, h, w])
            out[c] = np.where(np.isneginf(best), 0.0, best)
    else:
        counts = np.bincount(cells, minlength=n_cells) if mode == "mean" else None
        for c in range(C):
            acc = np.bincount(cells, weights=weights * features[n, c, h, w], minlength=n_cells)
            if counts is not None:
                acc = np.divide(acc, counts, out=np.zeros_like(acc), where=counts > 0)
            out[c] = acc
    return out


def reorder_weights(dist, ranks):
    """Restates pooling.py:258-261."""
    return np.ascontiguousarray(dist.transpose(0, 2, 3, 1)).reshape(-1)[ranks]


def prefixsum_pool(features, dist, ranks, starts, icells, n_cells, mode="sum"):
    """Restates pooling.py:162-196 (the LSS cumsum baseline)."""
    N, C, H, W = features.shape
    D = dist.shape[1]
    out = np.zeros((C, n_cells), dtype=np.float32)
    if starts.size == 0 or C == 0:
        return out
    r = ranks.astype(np.int64)
    d = r % D
    rest = r // D
    w = rest % W
    rest //= W
    h = rest % H
    n = rest // H
    weights = dist[n, d, h, w].astype(np.float64)
    bounds = np.append(starts.astype(np.int64), r.size)
    ends = bounds[1:] - 1
    lengths = np.diff(bounds)
    for c in range(C):
        running = np.cumsum(weights * features[n, c, h, w])
        seg = running[ends]
        seg[1:] -= running[ends[:-1]]
        if mode == "mean":
            seg /= lengths
        ch = np.zeros(n_cells)
        ch[icells.astype(np.int64)] = seg
        out[c] = ch
    return out


# --------------------------------------------------------------------------
# materialised lift and backward (no reference counterpart: SPEC.md:540
# lists autograd as a non-goal; these fp64 restatements define the math)
# --------------------------------------------------------------------------

def lift(features, dist):
    """x[(n,h,w,d), c] = dist[n,d,h,w] * features[n,c,h,w] in the reference
    point order (geometry.py:106-107); fp32 product."""
    f = features.transpose(0, 2, 3, 1)[:, :, :, None, :]   # N,H,W,1,C
    w = dist.transpose(0, 2, 3, 1)[:, :, :, :, None]       # N,H,W,D,1
    return np.ascontiguousarray((w * f).reshape(-1, features.shape[1]).astype(np.float32))


def pool_backward(features, dist, cell_of_point, grad_out, ranks, starts,
                  icells, mode="sum"):
    """fp64 gradient of pool_interval w.r.t. features and dist.

    grad_out: (C, n_cells).  SUM: dL/dv_p = g[:, cell(p)];  MEAN: scaled by
    1/len(cell);  MAX: routed to the first point (rank order) attaining the
    max, per channel.  Returns (grad_features (N,C,H,W), grad_dist (N,D,H,W))
    as float64."""
    N, C, H, W = features.shape
    D = dist.shape[1]
    n_cells = grad_out.shape[1]
    g = grad_out.astype(np.float64)
    P = N * H * W * D
    gv = np.zeros((P, C))                      # dL/d(value of point p)
    if mode in ("sum", "mean"):
        keep = cell_of_point != OUT_OF_RANGE
        cells = cell_of_point[keep].astype(np.int64)
        scale = np.ones(n_cells)
        if mode == "mean":
            counts = np.bincount(cells, minlength=n_cells)
            scale = np.where(counts > 0, 1.0 / np.maximum(counts, 1), 0.0)
        gv[keep] = (g[:, cells] * scale[cells]).T
    else:
        f_t = features.transpose(0, 2, 3, 1).reshape(-1, C).astype(np.float64)
        w_t = dist.transpose(0, 2, 3, 1).reshape(-1).astype(np.float64)
        bounds = np.append(starts.astype(np.int64), ranks.size)
        for i in range(starts.size):
            pts = ranks[bounds[i]:bounds[i + 1]].astype(np.int64)
            vals = w_t[pts, None] * f_t[pts // D]            # L x C
            arg = np.argmax(vals, axis=0)                     # first max
            gv[pts[arg], np.arange(C)] += g[:, int(icells[i])]
    gv = gv.reshape(N, H, W, D, C)
    f = features.astype(np.float64).transpose(0, 2, 3, 1)      # N,H,W,C
    wd = dist.astype(np.float64).transpose(0, 2, 3, 1)         # N,H,W,D
    grad_f = np.einsum("nhwdc,nhwd->nchw", gv, wd)
    grad_w = np.einsum("nhwdc,nhwc->ndhw", gv, f)
    return grad_f, grad_w


def bf16_round(a: np.ndarray) -> np.ndarray:
    """float32 -> nearest-even bfloat16 -> float32 (finite inputs)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).reshape(np.shape(a))


def fused_pool(features_bf16_as_f32, logits_bf16_as_f32, ranks, starts,
               icells, n_cells, mode="sum"):
    """Fused lift+pool semantics on bf16-rounded inputs: softmax over D
    (fp64) then the 64-bit interval reduction."""
    dist = normalize_depth(logits_bf16_as_f32)
    return pool_interval(features_bf16_as_f32, dist, ranks, starts, icells,
                         n_cells, mode)


def fused_backward(ctx_bf16_as_f32, logits_bf16_as_f32, cell_of_point, grad_out, ranks,
                   starts, icells, mode="sum"):
    """fp64 gradient of pool(softmax_D(logits) (x) context) (the fused path)
    w.r.t. logits and context: the pooling adjoint (pool_backward) on the
    fp64 softmax, then the softmax Jacobian
    dL/dl[d] = w[d] (dL/dw[d] - sum_d' w[d'] dL/dw[d']).
    Returns (grad_logits (N,D,H,W), grad_context (N,C,H,W)) as float64."""
    x = np.asarray(logits_bf16_as_f32, dtype=np.float64)
    e = np.exp(x - x.max(axis=1, keepdims=True))
    w = e / e.sum(axis=1, keepdims=True)
    gc, gw = pool_backward(ctx_bf16_as_f32, w, cell_of_point, grad_out, ranks, starts, icells,
                           mode)
    s = (w * gw).sum(axis=1, keepdims=True)
    return w * (gw - s), gc


def max_rel_dev(reference, candidate) -> float:
    """max |a-b| / max(1, |a|) -- the reference suite's metric
    (tests/conftest.py:68-74 of the reference)."""
    a = np.asarray(reference, dtype=np.float64)
    b = np.asarray(candidate, dtype=np.float64)
    if a.size == 0:
        return 0.0
    return float((np.abs(a - b) / np.maximum(1.0, np.abs(a))).max())


# --------------------------------------------------------------------------
# shared-BEV fusion (fusion.py) -- §8f "next" components
# --------------------------------------------------------------------------

def quantize_points(grid7, nx, ny, xyz):
    """Restates bevgrid.py:85-98 on float64 (M, 3) points."""
    x_min, _, y_min, _, z_min, z_max, r = grid7
    pts = np.asarray(xyz, dtype=np.float64)
    ix = np.floor((pts[:, 0] - x_min) / r).astype(np.int64)
    iy = np.floor((pts[:, 1] - y_min) / r).astype(np.int64)
    z = pts[:, 2]
    ok = (ix >= 0) & (ix < nx) & (iy >= 0) & (iy < ny) & (z >= z_min) & (z < z_max)
    return np.where(ok, ix * ny + iy, OUT_OF_RANGE).astype(np.uint32)


def lidar_to_bev(points, grid7, nx, ny, mode="sum"):
    """Restates fusion.py:19-53: (3, nx, ny) float32 count / intensity /
    height, fp64 bincount sums in input order."""
    points = np.asarray(points, dtype=np.float64)
    n_cells = nx * ny
    out = np.zeros((3, n_cells), dtype=np.float32)
    if points.shape[0]:
        cells = quantize_points(grid7, nx, ny, points[:, :3])
        keep = cells != OUT_OF_RANGE
        cells = cells[keep].astype(np.int64)
        counts = np.bincount(cells, minlength=n_cells)
        out[0] = counts
        for ch, values in ((1, points[keep, 3]), (2, points[keep, 2])):
            if mode == "max":
                best = np.full(n_cells, -np.inf)
                np.maximum.at(best, cells, values)
                out[ch] = np.where(np.isneginf(best), 0.0, best)
            else:
                acc = np.bincount(cells, weights=values, minlength=n_cells)
                if mode == "mean":
                    acc = np.divide(acc, counts, out=np.zeros_like(acc), where=counts > 0)
                out[ch] = acc
    return out.reshape(3, nx, ny)


def grid_resample(values, src7, src_nx, src_ny, dst7, dst_nx, dst_ny):
    """Restates fusion.py:70-108 (bilinear between cell centres, fp64)."""
    eps = 1e-9
    gx = (dst7[0] + (np.arange(dst_nx) + 0.5) * dst7[6] - src7[0]) / src7[6] - 0.5
    gy = (dst7[2] + (np.arange(dst_ny) + 0.5) * dst7[6] - src7[2]) / src7[6] - 0.5
    cov_x = (gx >= -eps) & (gx <= src_nx - 1 + eps)
    cov_y = (gy >= -eps) & (gy <= src_ny - 1 + eps)
    gx = np.clip(gx, 0.0, src_nx - 1)
    gy = np.clip(gy, 0.0, src_ny - 1)
    x0 = np.floor(gx).astype(np.int64)
    y0 = np.floor(gy).astype(np.int64)
    x1 = np.minimum(x0 + 1, src_nx - 1)
    y1 = np.minimum(y0 + 1, src_ny - 1)
    fx = np.clip(gx - x0, 0.0, 1.0)[None, :, None]
    fy = np.clip(gy - y0, 0.0, 1.0)[None, None, :]
    v = np.asarray(values).astype(np.float64)
    ix0, ix1 = x0[:, None], x1[:, None]
    iy0, iy1 = y0[None, :], y1[None, :]
    interp = (v[:, ix0, iy0] * (1 - fx) * (1 - fy) + v[:, ix1, iy0] * fx * (1 - fy)
              + v[:, ix0, iy1] * (1 - fx) * fy + v[:, ix1, iy1] * fx * fy)
    interp *= (cov_x[:, None] & cov_y[None, :])[None, :, :]
    return interp.astype(np.float32)
