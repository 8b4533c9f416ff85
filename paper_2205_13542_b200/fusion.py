"""Shared-BEV fusion on the GPU (reference fusion.py:1-117).

The camera pool's consumers: LiDAR flattening into the same BEV grid, channel
concatenation, bilinear resampling between grids, and the encoder hook.
``lidar_to_bev`` and ``grid_resample`` run in sm_100a kernels
(csrc/fusion.cu) and are bit-identical to the reference; numpy inputs give
numpy maps like the reference's, CUDA tensors stay on the device.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .bevgrid import BevGridSpec, cuda_device, ptr, stream_ptr, to_numpy
from .errors import ValidationError
from .pooling import _MODE, BevFeatureMap, Reducer, _reducer


def _host_or_device(values) -> tuple[torch.Tensor, bool]:
    if isinstance(values, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(values)), True
    if isinstance(values, torch.Tensor):
        return values, not values.is_cuda
    raise ValidationError("expected a numpy array or a torch tensor")


def lidar_to_bev(points, grid: BevGridSpec, reducer=Reducer.SUM) -> BevFeatureMap:
    """Flatten an (M, 4) LiDAR cloud (x, y, z, intensity) along z
    (fusion.py:19-53): channels point count, reduced intensity, reduced
    height.  The count ignores the reducer; points outside the grid
    contribute nothing; an empty cloud gives zeros."""
    reducer = _reducer(reducer)
    t, host = _host_or_device(points)
    if t.dim() != 2 or t.shape[1] != 4:
        raise ValidationError(f"expected an (M, 4) point array, got {tuple(t.shape)}")
    dev = cuda_device(None if host else t.device)
    t = t.to(dev, torch.float64).contiguous()
    if t.numel() and not bool(torch.isfinite(t).all()):
        raise ValidationError("point cloud contains non-finite values")
    M = int(t.shape[0])
    out = torch.empty((3, grid.n_cells), dtype=torch.float32, device=dev)
    ws = torch.empty(_lib.load().bvp_lidar_workspace_bytes(M, grid.nx, grid.ny),
                     dtype=torch.uint8, device=dev)
    g = grid.as_array()
    _lib.call("bvp_lidar_to_bev", ptr(t) if M else None, M, g.ctypes.data, grid.nx, grid.ny,
              _MODE[reducer], ptr(out), ptr(ws), ws.numel(), stream_ptr(dev))
    v = out.view(3, grid.nx, grid.ny)
    return BevFeatureMap(to_numpy(v) if host else v, grid)


def fuse_concat(a: BevFeatureMap, b: BevFeatureMap) -> BevFeatureMap:
    """Concatenate two BEV maps along channels, a's first (fusion.py:56-67).
    Both must live on the same grid.  Values are copied (a device copy for
    CUDA maps).  A camera map pooled straight into a channel slice of a
    preallocated buffer (PoolPlan.reduce(out=...)) avoids even that copy."""
    if a.grid != b.grid:
        raise ValidationError(
            "cannot concatenate maps on different grids; "
            "use grid_resample to bring one onto the other's grid")
    if isinstance(a.values, torch.Tensor) or isinstance(b.values, torch.Tensor):
        va = torch.as_tensor(a.values)
        vb = torch.as_tensor(b.values)
        dev = va.device if va.is_cuda else vb.device
        return BevFeatureMap(torch.cat([va.to(dev), vb.to(dev)], dim=0), a.grid)
    return BevFeatureMap(np.concatenate([a.values, b.values], axis=0), a.grid)


def grid_resample(src: BevFeatureMap, dst_grid: BevGridSpec) -> BevFeatureMap:
    """Bilinear resampling of a BEV map onto another grid (fusion.py:70-108):
    destination cell centres sample the four surrounding source centres;
    centres outside the source centre span give 0; z extents are ignored."""
    t, host = _host_or_device(src.values)
    if t.dim() != 3:
        raise ValidationError("expected a (C, nx, ny) map")
    sg = src.grid
    dev = cuda_device(None if host else t.device)
    t = t.to(dev, torch.float32).contiguous()
    C = int(t.shape[0])
    out = torch.empty((C, dst_grid.nx, dst_grid.ny), dtype=torch.float32, device=dev)
    sa, da = sg.as_array(), dst_grid.as_array()
    _lib.call("bvp_grid_resample_f32", ptr(t), C, sa.ctypes.data, sg.nx, sg.ny, da.ctypes.data,
              dst_grid.nx, dst_grid.ny, ptr(out), stream_ptr(dev))
    return BevFeatureMap(to_numpy(out) if host else out, dst_grid)


def bev_encoder(fused: BevFeatureMap) -> BevFeatureMap:
    """Stable call site for a BEV encoder; the identity, as in the reference
    (fusion.py:111-117)."""
    return fused
