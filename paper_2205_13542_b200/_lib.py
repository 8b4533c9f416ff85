"""ctypes binding of libbevpool_sm100.so (the C ABI in include/bevpool_b200.h).

There is deliberately no fallback: if the shared library is missing or fails
to load, every GPU entry point raises ``ExtensionMissingError`` -- the
framework never silently computes on the CPU.
"""

from __future__ import annotations

import ctypes
import os

from .errors import CudaError, ExtensionMissingError, from_status  # noqa: F401

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbevpool_sm100.so")

BVP_OK, BVP_ERR_INVALID, BVP_ERR_UNSUPPORTED, BVP_ERR_CUDA = 0, 1, 2, 3
BVP_SUM, BVP_MEAN, BVP_MAX, BVP_MEAN_DIV = 0, 1, 2, 3
TILE_CELLS = 32
OUT_OF_RANGE = 0xFFFFFFFF
BVP_OUT_ZEROED = 0x100  # include/bevpool_b200.h
BVP_TILE_PHASE1 = 0x200
BVP_TILE_PHASE2 = 0x400
ABI_VERSION = 9


_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_int64
_D = ctypes.c_double
_S = ctypes.c_size_t


class Schedule(ctypes.Structure):
    """struct bvp_schedule (include/bevpool_b200.h)."""
    _fields_ = [("point_meta", _P), ("work", _P), ("splits", _P), ("work_counts", _P),
                ("max_work", _L), ("max_splits", _L), ("max_partials", _L), ("chunk", _L)]


_SP = ctypes.POINTER(Schedule)


class TilePlanStruct(ctypes.Structure):
    """struct bvp_tile_plan (include/bevpool_b200.h)."""
    _fields_ = [("N", _I), ("H", _I), ("W", _I), ("D", _I), ("n_cells", _L), ("base", _P),
                ("bytes", _S), ("max_seg", _L), ("tile_rows", _I), ("n_tiles", _L),
                ("n_seg", _P), ("cell_seg_first", _P), ("cell_points", _P)]


_TP = ctypes.POINTER(TilePlanStruct)

#: name -> (restype, argtypes); mirrors include/bevpool_b200.h one to one
SIGNATURES = {
    "bvp_abi_version": (_I, []),
    "bvp_last_error": (ctypes.c_char_p, []),
    "bvp_frustum_cells": (_I, [_P, _I, _I, _I, _I, _D, _D, _P, _I, _I, _P, _P]),
    "bvp_frustum_points": (_I, [_P, _I, _I, _I, _I, _D, _D, _P, _P]),
    "bvp_quantize_points": (_I, [_P, _L, _P, _I, _I, _P, _P]),
    "bvp_interval_reduce_f32": (_I, [_P, _P, _P, _L, _L, _P, _P, _P, _L, _I, _I, _I, _I, _I, _P]),
    "bvp_depth_distribution_check": (_I, [_P, _I, _I, _I, _I, _P, _P]),
    "bvp_sort_workspace_bytes": (_S, [_L, _L]),
    "bvp_sort_intervals": (_I, [_P, _L, _L, _P, _P, _P, _P, _P, _P, _P, _S, _P]),
    "bvp_build_cache": (_I, [_P, _I, _I, _I, _I, _D, _D, _P, _I, _I, _P, _P, _P, _P, _P, _P,
                             _P, _P, _S, _P]),
    "bvp_build_association": (_I, [_P, _I, _I, _I, _I, _D, _D, _P, _I, _I, _P, _P, _P, _P, _P, _P,
                                   _P, _I, _P, _P, _P, _P, _P, _S, _P, _S, _P]),
    "bvp_pool_workspace_bytes": (_S, [_I, _I, _I, _I, _I]),
    "bvp_point_meta": (_I, [_P, _P, _I, _I, _I, _I, _P, _P]),
    "bvp_work_capacity": (_L, [_L, _L, _I]),
    "bvp_work_workspace_bytes": (_S, [_L, _L, _I, _I, _I, _I]),
    "bvp_make_work": (_I, [_P, _P, _P, _L, _L, _I, _I, _I, _I, _P, _P, _P, _P, _S, _P]),
    "bvp_pool_scratch_bytes": (_S, [_SP, _I, _I, _I]),
    "bvp_pool_forward_f32": (_I, [_P, _P, _P, _P, _P, _P, _SP, _I, _I, _I, _I, _I, _I, _I, _I,
                                  _L, _I, _I, _P, _P, _P, _P, _S, _P]),
    "bvp_pool_forward_nhwc_f32": (_I, [_P, _P, _P, _P, _P, _P, _SP, _I, _I, _I, _I, _I, _I, _I,
                                       _I, _L, _I, _I, _P, _P, _P, _S, _P]),
    "bvp_to_nhwc_f32": (_I, [_P, _I, _I, _I, _P, _P]),
    "bvp_pool_prepare_f32": (_I, [_P, _I, _I, _I, _I, _I, _P, _P, _L, _P]),
    "bvp_zero_empty_cells": (_I, [_P, _L, _I, _I, _P, _P]),
    "bvp_reorder_weights": (_I, [_P, _P, _L, _I, _I, _I, _I, _P, _P]),
    "bvp_normalize_depth": (_I, [_P, _I, _I, _I, _I, _P, _P]),
    "bvp_any_nonfinite": (_I, [_P, _L, _P, _P]),
    "bvp_lift_f32": (_I, [_P, _P, _I, _I, _I, _I, _I, _P, _P]),
    "bvp_pool_lifted_f32": (_I, [_P, _P, _P, _P, _P, _SP, _I, _I, _I, _I, _P, _P, _S, _P]),
    "bvp_fused_workspace_bytes": (_S, [_I, _I, _I, _I, _I, _I]),
    "bvp_fused_pool_bf16": (_I, [_P, _P, _P, _P, _P, _P, _SP, _I, _I, _I, _I, _I, _I, _I, _I,
                                 _I, _P, _P, _S, _P, _S, _P]),
    "bvp_backward_workspace_bytes": (_S, [_I, _I, _L]),
    "bvp_fused_backward_workspace_bytes": (_S, [_I, _I, _I, _I, _I, _I, _L]),
    "bvp_fused_backward_bf16": (_I, [_P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I,
                                     _L, _I, _P, _P, _P, _S, _P]),
    "bvp_pool_backward_f32": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I,
                                   _I, _L, _I, _P, _P, _P, _S, _P]),
    "bvp_pool_lifted_backward_f32": (_I, [_P, _P, _P, _P, _P, _I, _L, _I, _I, _L, _I, _P, _P,
                                          _S, _P]),
    "bvp_lidar_workspace_bytes": (_S, [_L, _I, _I]),
    "bvp_lidar_to_bev": (_I, [_P, _L, _P, _I, _I, _I, _P, _P, _S, _P]),
    "bvp_grid_resample_f32": (_I, [_P, _I, _P, _I, _I, _P, _I, _I, _P, _P]),
    "bvp_tile_plan_supported": (_I, [_I, _I, _I, _I, _L]),
    "bvp_tile_plan_bytes": (_S, [_I, _I, _I, _I, _L]),
    "bvp_tile_plan_workspace_bytes": (_S, [_I, _I, _I, _I, _L]),
    "bvp_tile_plan_init": (_I, [_TP, _I, _I, _I, _I, _L, _P, _S, _L]),
    "bvp_build_tile_plan": (_I, [_P, _TP, _P, _S, _P]),
    "bvp_build_tile_plan_ranks": (_I, [_P, _P, _P, _TP, _P, _S, _P]),
    "bvp_tile_backward_f32": (_I, [_P, _P, _P, _TP, _I, _I, _I, _P, _S, _P, _P, _P]),
    "bvp_tile_pool_f32": (_I, [_P, _P, _TP, _I, _I, _I, _P, _S, _P, _P]),
    "bvp_tile_pool_fused_bf16": (_I, [_P, _P, _TP, _I, _I, _I, _P, _S, _P, _P]),
    "bvp_tile_fused_backward_bf16": (_I, [_P, _P, _P, _TP, _I, _I, _I, _P, _S, _P, _P, _P]),
    "bvp_prefixsum_workspace_bytes": (_S, [_L, _I]),
    "bvp_pool_prefixsum_f32": (_I, [_P, _P, _P, _P, _P, _L, _L, _I, _I, _I, _I, _I, _L, _I, _P,
                                    _P, _S, _P]),
}

_lib = None


def load():
    """Load and type the library (once)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ExtensionMissingError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:  # pragma: no cover - depends on the box
        raise ExtensionMissingError(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.bvp_abi_version() != ABI_VERSION:
        raise ExtensionMissingError("libbevpool_sm100.so ABI version mismatch; rebuild it")
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if rc == BVP_OK:
        return
    raise from_status(rc, f"{what}: {load().bvp_last_error().decode(errors='replace')}")


#: per-entry-point call counts while a ``counting()`` block is active (the
#: analogue of the reference's debug.counting, debug.py:23-32: it proves the
#: cached forward launches no geometry)
_counts: dict | None = None


class counting:
    """Context manager: record how often each C entry point is called."""

    def __enter__(self) -> dict:
        global _counts
        self._prev = _counts
        _counts = {}
        return _counts

    def __exit__(self, *exc) -> None:
        global _counts
        _counts = self._prev


def call(name: str, *args) -> None:
    if _counts is not None:
        _counts[name] = _counts.get(name, 0) + 1
    check(getattr(load(), name)(*args), name)
