"""Depth distributions (reference lift.py:17-63), computed on the GPU."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .bevgrid import cuda_device, ptr, stream_ptr, to_numpy
from .errors import ValidationError


def nonfinite_flags(*tensors: torch.Tensor) -> list:
    """Device finiteness scans of float32 CUDA tensors, one flag each, read
    back with a single host sync."""
    if not tensors:
        return []
    flags = torch.zeros(len(tensors), dtype=torch.int32, device=tensors[0].device)
    for k, t in enumerate(tensors):
        t = t.contiguous()
        if t.numel():
            _lib.call("bvp_any_nonfinite", ptr(t), t.numel(), ptr(flags[k:]),
                      stream_ptr(t.device))
    return [bool(v) for v in flags.tolist()]


def any_nonfinite(t: torch.Tensor) -> bool:
    """Device finiteness scan of a float32 CUDA tensor (one host sync)."""
    return nonfinite_flags(t)[0]


def normalize_depth(logits, check_finite: bool = True):
    """Softmax over D of (N, D, H, W) (or (B, N, D, H, W)) logits.

    64-bit max-subtracted softmax stored float32, like the reference
    (lift.py:17-31).  numpy in -> numpy out (one H2D + D2H); CUDA tensor in
    -> CUDA tensor out.
    """
    host = isinstance(logits, np.ndarray)
    if host:
        if logits.ndim != 4:
            raise ValidationError(f"logits must be (N, D, H, W), got shape {logits.shape}")
        t = torch.from_numpy(np.ascontiguousarray(logits, dtype=np.float32)).to(cuda_device())
    else:
        t = logits
        if t.dim() not in (4, 5):
            raise ValidationError(f"logits must be (N, D, H, W), got shape {tuple(t.shape)}")
        if t.dtype != torch.float32:
            t = t.float()
        t = t.contiguous()
    if check_finite and any_nonfinite(t):
        raise ValidationError("logits contain non-finite values")
    *lead, D, H, W = t.shape
    NB = int(np.prod(lead))
    out = torch.empty_like(t)
    if t.numel():
        _lib.call("bvp_normalize_depth", ptr(t), NB, D, H, W, ptr(out), stream_ptr(t.device))
    return to_numpy(out) if host else out


def point_weight(dist, n: int, h: int, w: int, d: int) -> float:
    """Depth probability of frustum point (n, h, w, d) (scalar accessor)."""
    n_cams, n_bins, height, width = dist.shape
    for name, value, bound in (("camera", n, n_cams), ("row", h, height), ("col", w, width),
                               ("depth bin", d, n_bins)):
        if not 0 <= value < bound:
            raise IndexError(f"{name} index {value} out of range [0, {bound})")
    return float(dist[n, d, h, w])


def check_depth_distribution(dist, tol: float = 1e-6) -> None:
    """Raise ValidationError unless ``dist`` (N, D, H, W) holds per-pixel
    distributions: no negative entry, every pixel's D probabilities summing
    to 1 within ``tol`` (reference lift.py:52-63).  The scan runs on the
    GPU (bvp_depth_distribution_check, fp64 sums)."""
    if len(dist.shape) != 4:
        raise ValidationError(f"distribution must be (N, D, H, W), got {tuple(dist.shape)}")
    host = isinstance(dist, np.ndarray)
    t = (torch.from_numpy(np.ascontiguousarray(dist, dtype=np.float32)).to(cuda_device()) if host
         else dist.float().contiguous())
    N, D, H, W = (int(v) for v in t.shape)
    if t.numel() == 0:
        return
    stats = torch.zeros(2, dtype=torch.int64, device=t.device)
    _lib.call("bvp_depth_distribution_check", ptr(t), N, D, H, W, ptr(stats), stream_ptr(t.device))
    neg, dev_bits = stats.tolist()
    worst = float(np.array([dev_bits], dtype=np.int64).view(np.float64)[0])
    if neg:
        raise ValidationError("distribution has negative entries")
    if worst > tol:
        raise ValidationError(
            f"per-pixel depth probabilities must sum to 1 (worst deviation {worst:.3e})")
