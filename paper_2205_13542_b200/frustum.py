"""generate_frustum / FrustumPoints / quantize_points on the GPU.

Drop-ins for the reference's geometry.py:102-191 and bevgrid.py:85-98.  The
frustum is computed in fp64 with the reference's exact rounding (the
OpenBLAS dgemm FMA chain; csrc/geometry.cu ego_at) and lives
on the device; ``FrustumPoints.coords`` is the reference-typed read-only
(P, 3) float64 numpy view, copied to the host on first access.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .bevgrid import BevGridSpec, cuda_device, ptr, stream_ptr, to_numpy
from .errors import ConfigurationError, ValidationError
from .geometry import CameraCalibration, FrustumSpec, rig_rows


class FrustumPoints:
    """Ego-frame coordinates of every frustum point of a rig (geometry.py:102-122).

    Row ((n*H + h)*W + w)*D + d holds point (n, h, w, d).  ``d_coords`` is the
    (P, 3) float64 CUDA tensor; ``coords`` its host copy (read-only)."""

    def __init__(self, d_coords: torch.Tensor, n_cameras: int, spec: FrustumSpec):
        self.d_coords = d_coords
        self.n_cameras = n_cameras
        self.spec = spec
        self._host = None

    @property
    def coords(self) -> np.ndarray:
        if self._host is None:
            a = to_numpy(self.d_coords).copy()
            a.flags.writeable = False
            self._host = a
        return self._host

    def __len__(self) -> int:
        return int(self.d_coords.shape[0])

    def point_index(self, n: int, h: int, w: int, d: int) -> int:
        s = self.spec
        return ((n * s.height + h) * s.width + w) * s.depth_bins + d

    def __repr__(self) -> str:
        return f"FrustumPoints(n_cameras={self.n_cameras}, points={len(self)})"


def generate_frustum(rig: list[CameraCalibration], spec: FrustumSpec,
                     device=None) -> FrustumPoints:
    """Unproject every (pixel, depth bin) of every camera into ego space on
    the GPU -- bit-identical to the reference's generate_frustum."""
    cams = rig_rows(rig)  # raises ConfigurationError for an empty rig
    dev = cuda_device(device)
    P = len(rig) * spec.points_per_camera
    d_cams = torch.from_numpy(cams).to(dev)
    coords = torch.empty((P, 3), dtype=torch.float64, device=dev)
    _lib.call("bvp_frustum_points", ptr(d_cams), len(rig), spec.height, spec.width,
              spec.depth_bins, spec.depth_min, spec.depth_step, ptr(coords), stream_ptr(dev))
    return FrustumPoints(coords, len(rig), spec)


def quantize_points(spec: BevGridSpec, points):
    """Flat cell ids of (M, 3) ego points (bevgrid.py:85-98), 0xFFFFFFFF out
    of range.  numpy in -> uint32 numpy out; a float64 CUDA tensor (or
    FrustumPoints) in -> int32 CUDA tensor holding the uint32 bits."""
    if isinstance(points, FrustumPoints):
        points = points.d_coords
    host = not isinstance(points, torch.Tensor)
    if host:
        arr = np.array(points, dtype=np.float64, order="C")  # own, writable copy
        if arr.ndim != 2 or arr.shape[1] != 3:
            raise ValidationError(f"points must be (M, 3), got {arr.shape}")
        t = torch.from_numpy(arr).to(cuda_device())
    else:
        if points.dim() != 2 or points.shape[1] != 3 or not points.is_cuda:
            raise ValidationError("points must be an (M, 3) CUDA tensor")
        t = points.to(torch.float64).contiguous()
    M = int(t.shape[0])
    cells = torch.empty(M, dtype=torch.int32, device=t.device)
    if M:
        grid = spec.as_array()
        _lib.call("bvp_quantize_points", ptr(t), M, grid.ctypes.data, spec.nx, spec.ny,
                  ptr(cells), stream_ptr(t.device))
    return to_numpy(cells).view(np.uint32) if host else cells


def _check_spec(spec) -> None:
    if not isinstance(spec, BevGridSpec):
        raise ConfigurationError("spec must be a BevGridSpec")
