"""The reference's public view-transform API on the GPU (its __init__.py:7-57):
generate_frustum / FrustumPoints, quantize_points, check_depth_distribution,
pool_naive, set/get_parallelism, and the "no geometry in a cached forward"
property (reference pkg/tests/test_bench.py:72-83 via debug.counting)."""

import json
import os

import numpy as np
import pytest
import torch

import paper_2205_13542_b200 as bp
from conftest import sha
from oracle import oracle as o
from paper_2205_13542_b200 import _lib

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "golden_frustum.json")))


def test_every_reference_name_is_exported():
    import re
    names = ["AssociationCache", "BevGridSpec", "build_cache", "deserialize_cache", "load_cache",
             "quantize", "quantize_points", "save_cache", "serialize_cache", "validate_cache",
             "DEFAULT_GRID", "OUT_OF_RANGE", "BehindCameraError", "BevPoolError",
             "ConfigurationError", "FileFormatError", "StaleCacheError",
             "UnsupportedReducerError", "ValidationError", "bev_encoder", "fuse_concat",
             "grid_resample", "lidar_to_bev", "CameraCalibration", "FrustumPoints",
             "FrustumSpec", "depth_of_bin", "generate_frustum", "load_calibration",
             "parse_calibration", "project", "save_calibration", "unproject",
             "check_depth_distribution", "normalize_depth", "point_weight", "BACKENDS",
             "BevFeatureMap", "Reducer", "get_parallelism", "pool", "pool_interval",
             "pool_naive", "pool_prefixsum", "reorder_weights", "set_parallelism",
             "load_tensor", "save_tensor", "WorkloadSpec", "gen_workload", "standard_spec",
             "synthetic_rig"]  # reference pkg/src/bevpool/__init__.py:7-57
    assert [n for n in names if not hasattr(bp, n)] == []
    assert re.match(r"\d+\.\d+", bp.__version__)
    assert bp.BACKENDS == ("naive", "prefixsum", "interval")


def test_parallelism_knob():
    assert bp.set_parallelism(3) == 3
    assert bp.get_parallelism() == 3
    assert bp.set_parallelism(0) == (os.cpu_count() or 1)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["T", "S"])
def test_generate_frustum_bit_identical_to_reference(name):
    spec = bp.CONFIGS[name]
    rig = bp.synthetic_rig(spec.n_cameras, spec.frustum)
    pts = bp.generate_frustum(rig, spec.frustum)
    assert len(pts) == GOLD["configs"][name]["n_points"]
    assert sha(pts.coords.astype("<f8")) == GOLD["configs"][name]["coords"]
    cells = bp.quantize_points(spec.grid, pts.coords)
    assert sha(cells.astype("<u4")) == GOLD["configs"][name]["cells"]
    # device in, device out: the same bits
    dcells = bp.quantize_points(spec.grid, pts)
    np.testing.assert_array_equal(dcells.cpu().numpy().view(np.uint32), cells)
    # and the association's own cells
    cache = bp.build_cache(rig, spec.frustum, spec.grid)
    np.testing.assert_array_equal(cells, cache.cell_of_point)


@pytest.mark.gpu
def test_frustum_matches_scalar_unproject_and_regenerates():
    """reference pkg/tests/test_geometry.py:141-164: every point equals the
    scalar unproject within 1e-12; regeneration is bit-identical."""
    rng = np.random.default_rng(7)
    spec = bp.FrustumSpec(5, 7, 1.0, 0.75, 9)
    rig = []
    for k in range(2):
        a, b = rng.uniform(-0.3, 0.3, 2)
        rz = np.array([[np.cos(a), -np.sin(a), 0], [np.sin(a), np.cos(a), 0], [0, 0, 1]])
        rx = np.array([[1, 0, 0], [0, np.cos(b), -np.sin(b)], [0, np.sin(b), np.cos(b)]])
        base = np.array([[0.0, 0.0, 1.0], [-1.0, 0.0, 0.0], [0.0, -1.0, 0.0]])
        rig.append(bp.CameraCalibration(6.0, 6.5, 3.1, 2.2, rz @ rx @ base,
                                        rng.uniform(-1, 1, 3), k))
    pts = bp.generate_frustum(rig, spec)
    for n, cam in enumerate(rig):
        for h in range(spec.height):
            for w in range(spec.width):
                for d in range(spec.depth_bins):
                    want = bp.unproject(cam, w, h, bp.depth_of_bin(spec, d))
                    got = pts.coords[pts.point_index(n, h, w, d)]
                    assert np.abs(got - want).max() <= 1e-12
    again = bp.generate_frustum(rig, spec)
    assert again.coords.tobytes() == pts.coords.tobytes()
    assert not pts.coords.flags.writeable
    with pytest.raises(bp.ConfigurationError):
        bp.generate_frustum([], spec)


@pytest.mark.gpu
def test_quantize_points_kats():
    """reference pkg/tests/test_bevgrid.py:48-73 KATs, evaluated by the
    reference (tests/golden/golden_frustum.json)."""
    got = bp.quantize_points(bp.DEFAULT_GRID, np.array(GOLD["kat"]["points"]))
    assert got.dtype == np.uint32
    assert got.tolist() == GOLD["kat"]["cells"]
    assert got[0] == 32896 and got[1] == bp.OUT_OF_RANGE and got[2] == 0
    for p, c in zip(GOLD["kat"]["points"], got):
        assert bp.quantize(bp.DEFAULT_GRID, p) == c
    assert bp.quantize_points(bp.DEFAULT_GRID, np.empty((0, 3))).shape == (0,)
    with pytest.raises(bp.ValidationError):
        bp.quantize_points(bp.DEFAULT_GRID, np.zeros((4, 2)))


@pytest.mark.gpu
def test_check_depth_distribution():
    """reference pkg/tests/test_lift.py: a softmax passes, negative entries and
    sums away from 1 raise ValidationError; CUDA tensors work too."""
    _, _, logits, _ = bp.gen_workload(bp.CONFIGS["T"])
    dist = bp.normalize_depth(logits)
    bp.check_depth_distribution(dist)
    bp.check_depth_distribution(torch.from_numpy(dist).cuda())
    bad = dist.copy()
    bad[0, 3, 2, 1] = -1e-3
    with pytest.raises(bp.ValidationError, match="negative"):
        bp.check_depth_distribution(bad)
    off = dist.copy()
    off[0, :, 4, 4] *= 1.01
    with pytest.raises(bp.ValidationError, match="sum to 1"):
        bp.check_depth_distribution(off)
    bp.check_depth_distribution(off, tol=0.02)
    with pytest.raises(bp.ValidationError):
        bp.check_depth_distribution(dist[0])


@pytest.mark.gpu
@pytest.mark.parametrize("red", ["sum", "mean", "max"])
def test_pool_naive_is_the_reference_scatter(red):
    """pool_naive (pooling.py:135-159): fp64 per-cell sums in point order,
    MEAN = sum / count; the numpy restatement of the reference's bincount
    scatter gives the same bits."""
    spec = bp.CONFIGS["T"]
    rig, features, logits, grid = bp.gen_workload(spec)
    cache = bp.build_cache(rig, spec.frustum, grid)
    dist = o.normalize_depth(logits)
    got = bp.pool_naive(features, dist, cache, grid, red).values
    want = o.pool_naive(features, dist, cache.cell_of_point, grid.n_cells, red)
    np.testing.assert_array_equal(got.reshape(want.shape), want)
    via = bp.pool(features, dist, cache, grid, red, backend="naive").values
    np.testing.assert_array_equal(via, got)


@pytest.mark.gpu
def test_cached_forward_launches_no_geometry():
    """reference pkg/tests/test_bench.py:72-83: the cold build projects and
    quantises (geometry entry points run), the cached forward does not."""
    spec = bp.CONFIGS["T"]
    rig, features, logits, grid = bp.gen_workload(spec)
    with _lib.counting() as cold:
        cache = bp.build_cache(rig, spec.frustum, grid)
    assert cold.get("bvp_build_cache", 0) == 1
    dist = bp.normalize_depth(logits)
    bp.pool_interval(features, dist, cache, grid)  # first use builds the tile plan
    geometry = ("bvp_frustum", "bvp_build", "bvp_sort", "bvp_quantize", "bvp_make", "bvp_point")
    for _ in range(2):
        with _lib.counting() as warm:
            bp.pool_interval(features, dist, cache, grid)
            bp.reorder_weights(dist, cache)
        assert not [k for k in warm if k.startswith(geometry)], warm
        assert warm.get("bvp_tile_pool_f32") == 1
