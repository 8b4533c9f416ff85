"""The reference-side binding: register this package as a ``"cuda"`` backend
of the reference's own pooling dispatch (pooling.py:52, :224-240).

    import bevpool                                  # the reference
    from examples.ref_backend_cuda import register
    register(bevpool)                               # adds backend "cuda"
    bevpool.pool(features, dist, cache, grid, bevpool.Reducer.SUM, backend="cuda")

The backend has the reference signature fn(features, dist, cache, grid,
reducer) -> BevFeatureMap.  It takes the reference's
AssociationCache as is: its cell_of_point goes to the GPU once per cache
(the sort, interval tables and tile plan are rebuilt there, bit-identical to
the cache's own), every call then pools on the B200.  ``exact=True`` gives
the reference's interval_reduce bits; the default fast mode is within 1e-5.
This file is what INTEGRATION.md §2 describes; tests/test_ref_host.py
executes it against the installed reference.
"""

from __future__ import annotations

import weakref

import numpy as np

import paper_2205_13542_b200 as bp

_caches: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _device_cache(cache, grid):
    """This package's device cache for a reference AssociationCache."""
    dc = _caches.get(cache)
    if dc is None:
        dc = bp.cache_from_cells(cache.cell_of_point, grid.nx, grid.ny, cache.fingerprint)
        _caches[cache] = dc
    return dc


def make_backend(ref, exact: bool = False):
    def pool_cuda(features, dist, cache, grid, reducer=ref.Reducer.SUM):
        ref.pooling._check_inputs(features, dist, cache, grid)  # reference validation
        g = bp.BevGridSpec(grid.x_min, grid.x_max, grid.y_min, grid.y_max, grid.z_min,
                           grid.z_max, grid.r)
        out = bp.pool_interval(np.asarray(features, np.float32), np.asarray(dist, np.float32),
                               _device_cache(cache, grid), g, str(reducer.value), exact=exact,
                               check_finite=False)
        return ref.BevFeatureMap(out.values, grid)
    return pool_cuda


def register(ref, name: str = "cuda", exact: bool = False) -> None:
    """Add the backend to the reference's dispatch table."""
    ref.pooling._BACKEND_FN[name] = make_backend(ref, exact)
    if name not in ref.pooling.BACKENDS:
        ref.pooling.BACKENDS = tuple(ref.pooling.BACKENDS) + (name,)


def register_kernel(ref) -> None:
    """Replace the reference's native kernel itself: _kernels.interval_reduce
    (_kernels.py:22-63) becomes a ctypes call of bvp_interval_reduce_f32 with
    the very same arguments -- the reference's pool_interval then runs its
    reduction on the GPU, bit for bit (out is written in place)."""
    import torch

    from paper_2205_13542_b200 import _lib
    from paper_2205_13542_b200.bevgrid import ptr, stream_ptr

    def interval_reduce(ranks, starts, interval_cells, dist_t, feats_t, out, height, width,
                        depth_bins, mode):
        dev = torch.device("cuda")
        t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in
             (("r", ranks.view(np.int32)), ("s", starts.view(np.int32)),
              ("c", interval_cells.view(np.int32)), ("d", dist_t), ("f", feats_t), ("o", out))}
        C, n_cells = out.shape
        _lib.call("bvp_interval_reduce_f32", ptr(t["r"]), ptr(t["s"]), ptr(t["c"]), len(ranks),
                  len(starts), ptr(t["d"]), ptr(t["f"]), ptr(t["o"]), n_cells, height, width,
                  depth_bins, C, int(mode), stream_ptr(dev))
        out[...] = t["o"].cpu().numpy()

    ref._kernels.interval_reduce = interval_reduce
