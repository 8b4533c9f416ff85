"""GPU parity: the CUDA path (through the C ABI) against the reference's own
outputs (golden SHA-256 digests) and the CPU oracle.

Bars (BASELINE.json north_star): cell ids / ranks / interval tables
bit-exact; pooled features bit-exact in exact (64-bit) mode and within 1e-5
(max |a-b| / max(1,|a|)) in fast fp32 mode; 1e-2 for the bf16 fused path.
"""

import numpy as np
import pytest
import torch

import paper_2205_13542_b200 as bp
from conftest import max_rel_dev, sha
from instances import GOLDEN_INSTANCES, random_instance
from oracle import oracle as o

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5
BF16_TOL = 1e-2


def rig_of(cams):
    return [bp.CameraCalibration(fx=r[0], fy=r[1], cx=r[2], cy=r[3], rotation=r[4:13].reshape(3, 3),
                                 translation=r[13:16], camera_id=k) for k, r in enumerate(cams)]


def specs_of(inst):
    frustum = bp.FrustumSpec(inst.height, inst.width, inst.depth_min, inst.depth_step,
                             inst.depth_bins)
    return frustum, bp.BevGridSpec(*inst.grid)


def check_against_golden(entry, cache, features, dist_np, grid, exact_pools=True):
    assert cache.n_in_range == entry["n_in"]
    assert cache.n_intervals == entry["n_int"]
    h = entry["sha256"]
    assert sha(cache.cell_of_point.astype("<u4")) == h["cell_of_point"]
    assert sha(cache.ranks.astype("<u4")) == h["ranks"]
    assert sha(cache.interval_starts.astype("<u4")) == h["interval_starts"]
    assert sha(cache.interval_cells.astype("<u4")) == h["interval_cells"]
    if exact_pools:
        for red in bp.Reducer:
            out = bp.pool_interval(features, dist_np, cache, grid, red, exact=True)
            assert sha(out.values.astype("<f4")) == h[f"pool_{red.value}"], red


# ---- geometry + sort + exact pooling, bit-exact vs the reference ----------

@pytest.mark.parametrize("name", ["T", "S", "H"])
def test_config_bit_exact_vs_reference(golden, name):
    spec = bp.CONFIGS[name]
    rig, features, logits, grid = bp.gen_workload(spec)
    cache = bp.build_cache(rig, spec.frustum, grid)
    dist = o.normalize_depth(logits)  # reference-identical weights
    check_against_golden(golden["configs"][name], cache, features, dist, grid)


@pytest.mark.parametrize("seed,mhw,md,mc", GOLDEN_INSTANCES)
def test_instances_bit_exact_vs_reference(golden, seed, mhw, md, mc):
    inst = random_instance(seed, mhw, md, mc)
    frustum, grid = specs_of(inst)
    cache = bp.build_cache(rig_of(inst.cams), frustum, grid)
    check_against_golden(golden["instances"][str(seed)], cache, inst.features,
                         o.normalize_depth(inst.logits), grid)


@pytest.mark.parametrize("name", ["T", "S"])
def test_fast_mode_within_tolerance(name):
    spec = bp.CONFIGS[name]
    rig, features, logits, grid = bp.gen_workload(spec)
    cache = bp.build_cache(rig, spec.frustum, grid)
    dist = o.normalize_depth(logits)
    for red in bp.Reducer:
        want = o.pool_interval(features, dist, cache.ranks, cache.interval_starts,
                               cache.interval_cells, grid.n_cells, red.value)
        got = bp.pool_interval(features, dist, cache, grid, red, exact=False)
        assert max_rel_dev(want, got.values.reshape(want.shape)) <= FP32_TOL, red


@pytest.mark.parametrize("seed", [10_000 + s for s in range(6)] + [100, 101, 300])
def test_fast_mode_random_instances(seed):
    inst = random_instance(seed, 64, 32, 16)
    frustum, grid = specs_of(inst)
    cache = bp.build_cache(rig_of(inst.cams), frustum, grid)
    dist = o.normalize_depth(inst.logits)
    for red in bp.Reducer:
        want = o.pool_naive(inst.features, dist, cache.cell_of_point, grid.n_cells, red.value)
        got = bp.pool_interval(inst.features, dist, cache, grid, red, exact=False)
        assert max_rel_dev(want, got.values.reshape(want.shape)) <= FP32_TOL


def test_normalize_depth_matches_reference(golden):
    for name in ("T", "S"):
        spec = bp.CONFIGS[name]
        _, _, logits, _ = bp.gen_workload(spec)
        got = bp.normalize_depth(logits)
        want = o.normalize_depth(logits)
        assert np.abs(got.astype(np.float64) - want).max() <= 1e-7
        assert (got == want).mean() > 0.999


# ---- reference KATs (test_pooling.py:141-183, test_bevgrid.py:77-172) ------

def worked_example():
    frustum = bp.FrustumSpec(1, 4, depth_min=1.0, depth_step=1.0, depth_bins=1)
    grid = bp.BevGridSpec(0.0, 1.2, 0.0, 0.4, -1, 1, r=0.4)
    cache = bp.cache_from_cells(np.array([2, 0, 2, 1], np.uint32), grid.nx, grid.ny, 0, 1,
                                frustum, grid)
    features = np.array([1, 2, 3, 4], np.float32).reshape(1, 1, 1, 4)
    dist = np.ones((1, 1, 1, 4), np.float32)
    return features, dist, cache, grid


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("red,want", [("sum", [2, 4, 4]), ("mean", [2, 4, 2]), ("max", [2, 4, 3])])
def test_worked_example(red, want, exact):
    f, d, cache, grid = worked_example()
    np.testing.assert_array_equal(cache.ranks, [1, 3, 0, 2])
    np.testing.assert_array_equal(cache.interval_starts, [0, 1, 2])
    np.testing.assert_array_equal(cache.interval_cells, [0, 1, 2])
    out = bp.pool(f, d, cache, grid, bp.Reducer(red), exact=exact)
    np.testing.assert_array_equal(out.values.reshape(3), want)


@pytest.mark.parametrize("red", ["sum", "mean"])
def test_prefixsum_backend(red):
    f, d, cache, grid = worked_example()
    out = bp.pool(f, d, cache, grid, bp.Reducer(red), backend="prefixsum")
    np.testing.assert_array_equal(out.values.reshape(3), [2, 4, 4] if red == "sum" else [2, 4, 2])
    inst = random_instance(10_003, 64, 32, 16)
    frustum, grid = specs_of(inst)
    cache = bp.build_cache(rig_of(inst.cams), frustum, grid)
    dist = o.normalize_depth(inst.logits)
    want = o.pool_naive(inst.features, dist, cache.cell_of_point, grid.n_cells, red)
    got = bp.pool(inst.features, dist, cache, grid, bp.Reducer(red), backend="prefixsum")
    assert max_rel_dev(want, got.values.reshape(want.shape)) < 1e-4


def test_one_hot_distribution_places_full_feature():
    rotation = np.column_stack([[0.0, -1.0, 0.0], [-1.0, 0.0, 0.0], [0.0, 0.0, -1.0]])
    cam = bp.CameraCalibration(fx=1, fy=1, cx=0, cy=0, rotation=rotation,
                               translation=np.array([0.2, 0.2, 4.0]))
    frustum = bp.FrustumSpec(1, 1, depth_min=0.5, depth_step=0.5, depth_bins=6)
    grid = bp.BevGridSpec(-2, 2, -2, 2, -5, 5, r=0.4)
    cache = bp.build_cache([cam], frustum, grid)
    assert cache.n_intervals == 1 and cache.n_in_range == 6
    assert int(cache.interval_cells[0]) == bp.quantize(grid, (0.2, 0.2, 0.0))
    features = np.full((1, 3, 1, 1), 7.5, np.float32)
    dist = np.zeros((1, 6, 1, 1), np.float32)
    dist[0, 2, 0, 0] = 1.0
    for backend in bp.BACKENDS:
        flat = bp.pool(features, dist, cache, grid, bp.Reducer.SUM, backend).values.reshape(3, -1)
        np.testing.assert_allclose(flat[:, int(cache.interval_cells[0])], 7.5, atol=1e-6)
        assert np.count_nonzero(flat) == 3


@pytest.mark.parametrize("backend", bp.BACKENDS)
def test_zero_weights_give_zero_map(backend):
    f, d, cache, grid = worked_example()
    assert not bp.pool(f, np.zeros_like(d), cache, grid, bp.Reducer.SUM, backend).values.any()


@pytest.mark.parametrize("backend", bp.BACKENDS)
def test_empty_ranks_give_zero_map(backend):
    frustum = bp.FrustumSpec(1, 4, 1.0, 1.0, 1)
    grid = bp.BevGridSpec(0.0, 1.2, 0.0, 0.4, -1, 1, r=0.4)
    cache = bp.cache_from_cells(np.full(4, bp.OUT_OF_RANGE, np.uint32), grid.nx, grid.ny, 0, 1,
                                frustum, grid)
    assert cache.n_in_range == 0 and cache.n_intervals == 0
    out = bp.pool(np.ones((1, 2, 1, 4), np.float32), np.ones((1, 1, 1, 4), np.float32), cache,
                  grid, bp.Reducer.SUM, backend)
    assert out.values.shape == (2, 3, 1) and not out.values.any()


@pytest.mark.parametrize("backend", bp.BACKENDS)
def test_zero_channels(backend):
    inst = random_instance(17)
    frustum, grid = specs_of(inst)
    cache = bp.build_cache(rig_of(inst.cams), frustum, grid)
    out = bp.pool(inst.features[:, :0], o.normalize_depth(inst.logits), cache, grid,
                  bp.Reducer.SUM, backend)
    assert out.values.shape == (0, grid.nx, grid.ny)


def test_all_points_out_of_range():
    inst = random_instance(0)
    frustum, _ = specs_of(inst)
    tiny = bp.BevGridSpec(1000, 1001, 1000, 1001, -1, 1, r=1.0)
    cache = bp.build_cache(rig_of(inst.cams), frustum, tiny)
    assert cache.n_in_range == 0 and cache.n_intervals == 0


def test_bit_identical_rebuild_and_rerun():
    spec = bp.CONFIGS["S"]
    rig, features, logits, grid = bp.gen_workload(spec)
    a = bp.build_cache(rig, spec.frustum, grid)
    b = bp.build_cache(rig, spec.frustum, grid)
    assert bp.serialize_cache(a) == bp.serialize_cache(b)
    dist = o.normalize_depth(logits)
    for exact in (True, False):
        x = bp.pool_interval(features, dist, a, grid, exact=exact).values
        y = bp.pool_interval(features, dist, a, grid, exact=exact).values
        assert x.tobytes() == y.tobytes()


def test_cache_round_trip(tmp_path):
    inst = random_instance(9)
    frustum, grid = specs_of(inst)
    rig = rig_of(inst.cams)
    cache = bp.build_cache(rig, frustum, grid)
    path = tmp_path / "cache.bvpc"
    bp.save_cache(path, cache)
    loaded = bp.load_cache(path)
    assert loaded.fingerprint == cache.fingerprint
    np.testing.assert_array_equal(loaded.ranks, cache.ranks)
    assert bp.validate_cache(loaded, rig, frustum, grid)
    dist = o.normalize_depth(inst.logits)
    a = bp.pool_interval(inst.features, dist, cache, grid).values
    b = bp.pool_interval(inst.features, dist, loaded, grid).values
    assert a.tobytes() == b.tobytes()


def test_reorder_weights_matches_rank_order():
    inst = random_instance(40)
    frustum, grid = specs_of(inst)
    cache = bp.build_cache(rig_of(inst.cams), frustum, grid)
    dist = o.normalize_depth(inst.logits)
    w = bp.reorder_weights(dist, cache)
    np.testing.assert_array_equal(w, o.reorder_weights(dist, cache.ranks))


class TestErrors:
    def test_unknown_backend(self):
        f, d, cache, grid = worked_example()
        with pytest.raises(bp.ConfigurationError, match="backend"):
            bp.pool(f, d, cache, grid, bp.Reducer.SUM, "gpu")

    def test_prefixsum_rejects_max(self):
        f, d, cache, grid = worked_example()
        with pytest.raises(bp.UnsupportedReducerError):
            bp.pool(f, d, cache, grid, bp.Reducer.MAX, "prefixsum")

    def test_shape_dtype_finite(self):
        f, d, cache, grid = worked_example()
        with pytest.raises(bp.ValidationError):
            bp.pool_interval(f[:, :, :, :2], d, cache, grid)
        with pytest.raises(bp.ValidationError, match="float32"):
            bp.pool_interval(f.astype(np.float64), d, cache, grid)
        bad = f.copy()
        bad[0, 0, 0, 0] = np.nan
        with pytest.raises(bp.ValidationError, match="finite"):
            bp.pool_interval(bad, d, cache, grid)

    def test_stale_cache(self):
        f, d, cache, grid = worked_example()
        with pytest.raises(bp.StaleCacheError):
            bp.pool_interval(np.ones((1, 1, 1, 5), np.float32), np.ones((1, 1, 1, 5), np.float32),
                             cache, grid)
        with pytest.raises(bp.StaleCacheError):
            bp.pool_interval(f, d, cache, bp.BevGridSpec(0.0, 2.4, 0.0, 0.8, -1, 1, r=0.4))


# ---- device tensors, batching, materialised and fused paths ---------------

def _S():
    spec = bp.CONFIGS["S"]
    rig, features, logits, grid = bp.gen_workload(spec)
    cache = bp.build_cache(rig, spec.frustum, grid)
    return spec, features, logits, grid, cache


def test_batched_device_pool_matches_per_sample():
    spec, features, logits, grid, cache = _S()
    dev = torch.device("cuda")
    feats = []
    dists = []
    for seed in range(3):
        _, f, lg, _ = bp.gen_workload(bp.WorkloadSpec(6, spec.frustum, grid, 80, seed))
        feats.append(torch.from_numpy(f))
        dists.append(torch.from_numpy(o.normalize_depth(lg)))
    F = torch.stack(feats).to(dev)
    Dd = torch.stack(dists).to(dev)
    out = bp.pool_interval(F, Dd, cache, grid, exact=True).values
    assert out.shape == (3, 80, grid.nx, grid.ny)
    for b in range(3):
        one = bp.pool_interval(F[b], Dd[b], cache, grid, exact=True).values
        assert torch.equal(out[b], one)


def test_materialised_lift_and_pool():
    spec, features, logits, grid, cache = _S()
    dist = o.normalize_depth(logits)
    dev = torch.device("cuda")
    x = bp.lift_features(torch.from_numpy(features).to(dev), torch.from_numpy(dist).to(dev))
    assert x.shape == (cache.n_points, 80)
    # lift is an exact fp32 product: spot-check rows against the oracle
    rows = np.random.default_rng(0).choice(cache.n_points, 4096, replace=False)
    want_x = o.lift(features, dist)[rows]
    np.testing.assert_array_equal(x[torch.from_numpy(rows).to(dev)].cpu().numpy(), want_x)
    for red in bp.Reducer:
        got = bp.pool_lifted(x, cache, grid, red).values.cpu().numpy()
        want = o.pool_interval(features, dist, cache.ranks, cache.interval_starts,
                               cache.interval_cells, grid.n_cells, red.value)
        assert max_rel_dev(want, got.reshape(want.shape)) <= FP32_TOL


def test_fused_bf16_path():
    spec, features, logits, grid, cache = _S()
    dev = torch.device("cuda")
    ctx = torch.from_numpy(features).to(dev).to(torch.bfloat16)
    lg = torch.from_numpy(logits).to(dev).to(torch.bfloat16)
    fb = o.bf16_round(features)
    lb = o.bf16_round(logits)
    for red in bp.Reducer:
        got = bp.pool_fused(lg, ctx, cache, grid, red).values.cpu().numpy().reshape(80, -1)
        # tight: same bf16 inputs, fp64 oracle
        want_b = o.fused_pool(fb, lb, cache.ranks, cache.interval_starts, cache.interval_cells,
                              grid.n_cells, red.value)
        assert max_rel_dev(want_b, got) <= 1e-5, red
        # the north-star bar: vs the fp32 reference path on unrounded inputs
        want = o.pool_interval(features, o.normalize_depth(logits), cache.ranks,
                               cache.interval_starts, cache.interval_cells, grid.n_cells,
                               red.value)
        assert max_rel_dev(want, got) <= BF16_TOL, red


def test_cache_builder_no_sync_rebuild_matches():
    spec, features, logits, grid, cache = _S()
    rig, _, _, _ = bp.gen_workload(spec)
    builder = bp.CacheBuilder(6, spec.frustum, grid)
    cams = torch.from_numpy(bp.rig_rows(rig)).cuda()
    for _ in range(2):
        c2 = builder.build(cams)
        torch.cuda.synchronize()
        assert c2.n_intervals == cache.n_intervals
        np.testing.assert_array_equal(c2.ranks, cache.ranks)
        c2._host_counts = None
        c2._host.clear()


# ---- gather backward (config B) vs the fp64 restatement --------------------

def _backward_case(name="T", seed=0):
    spec = bp.CONFIGS[name]
    rig, features, logits, grid = bp.gen_workload(bp.WorkloadSpec(
        spec.n_cameras, spec.frustum, spec.grid, spec.channels, seed))
    cache = bp.build_cache(rig, spec.frustum, grid)
    dist = o.normalize_depth(logits)
    g = np.random.default_rng(seed + 7).normal(size=(features.shape[1], grid.n_cells))
    return spec, features, dist, grid, cache, g.astype(np.float32)


@pytest.mark.parametrize("red", ["sum", "mean", "max"])
def test_backward_matches_fp64_restatement(red):
    spec, features, dist, grid, cache, g = _backward_case("T")
    dev = torch.device("cuda")
    f = torch.from_numpy(features).to(dev).requires_grad_(True)
    d = torch.from_numpy(dist).to(dev).requires_grad_(True)
    out = bp.bev_pool(f, d, cache, grid, red)
    want_out = o.pool_interval(features, dist, cache.ranks, cache.interval_starts,
                               cache.interval_cells, grid.n_cells, red)
    assert max_rel_dev(want_out, out.detach().cpu().numpy().reshape(want_out.shape)) <= FP32_TOL
    out.backward(torch.from_numpy(g).to(dev).view_as(out))
    gf, gw = o.pool_backward(features, dist, cache.cell_of_point, g.astype(np.float64),
                             cache.ranks, cache.interval_starts, cache.interval_cells, red)
    assert max_rel_dev(gf, f.grad.cpu().numpy()) <= FP32_TOL
    assert max_rel_dev(gw, d.grad.cpu().numpy()) <= FP32_TOL


def test_backward_batched_matches_per_sample():
    spec, features, dist, grid, cache, g = _backward_case("T")
    dev = torch.device("cuda")
    _, f2, l2, _ = bp.gen_workload(bp.WorkloadSpec(spec.n_cameras, spec.frustum, grid,
                                                   spec.channels, 1))
    F = torch.from_numpy(np.stack([features, f2])).to(dev).requires_grad_(True)
    Dd = torch.from_numpy(np.stack([dist, o.normalize_depth(l2)])).to(dev).requires_grad_(True)
    G = torch.from_numpy(np.stack([g, -g])).to(dev).view(2, spec.channels, grid.nx, grid.ny)
    bp.bev_pool(F, Dd, cache, grid).backward(G)
    for b in range(2):
        fb = F[b].detach().clone().requires_grad_(True)
        db = Dd[b].detach().clone().requires_grad_(True)
        bp.bev_pool(fb, db, cache, grid).backward(G[b])
        assert torch.equal(fb.grad, F.grad[b])
        assert torch.equal(db.grad, Dd.grad[b])


def test_backward_nuscenes_shape_sum():
    """SUM gradients at the S shape, restated per camera in fp64 (the full
    (P, C) fp64 oracle would need 1.3 GB)."""
    spec, features, dist, grid, cache, g = _backward_case("S")
    dev = torch.device("cuda")
    f = torch.from_numpy(features).to(dev).requires_grad_(True)
    d = torch.from_numpy(dist).to(dev).requires_grad_(True)
    bp.bev_pool(f, d, cache, grid).backward(torch.from_numpy(g).to(dev).view(80, grid.nx, grid.ny))
    N, C, H, W = features.shape
    D = dist.shape[1]
    cells = cache.cell_of_point.reshape(N, H, W, D)
    g64 = np.concatenate([g.astype(np.float64), np.zeros((C, 1))], axis=1)  # OOR -> zero column
    gf_got, gw_got = f.grad.cpu().numpy(), d.grad.cpu().numpy()
    for n in range(N):
        idx = np.where(cells[n] == bp.OUT_OF_RANGE, grid.n_cells, cells[n]).astype(np.int64)
        gc = g64[:, idx]                                   # C, H, W, D
        gf = np.einsum("chwd,dhw->chw", gc, dist[n].astype(np.float64))
        gw = np.einsum("chwd,chw->dhw", gc, features[n].astype(np.float64))
        assert max_rel_dev(gf, gf_got[n]) <= FP32_TOL
        assert max_rel_dev(gw, gw_got[n]) <= FP32_TOL


# ---- lane layouts: every channel count the fast kernels instantiate --------

def _sweep_case(C, seed=7):
    spec = bp.CONFIGS["T"]
    rng = np.random.default_rng(seed)
    rig, _, logits, grid = bp.gen_workload(spec)
    cache = bp.build_cache(rig, spec.frustum, grid)
    features = rng.uniform(-1, 1, size=(1, C, spec.frustum.height, spec.frustum.width)
                           ).astype(np.float32)
    return cache, grid, features, logits


@pytest.mark.parametrize("C", [1, 3, 4, 8, 12, 20, 33, 64, 80, 96, 128, 200, 256])
@pytest.mark.parametrize("red", ["sum", "mean", "max"])
def test_fast_mode_channel_sweep(C, red):
    cache, grid, features, logits = _sweep_case(C)
    dist = o.normalize_depth(logits)
    want = o.pool_interval(features, dist, cache.ranks, cache.interval_starts,
                           cache.interval_cells, grid.n_cells, red)
    got = bp.pool_interval(features, dist, cache, grid, red, exact=False).values
    assert max_rel_dev(want, got.reshape(want.shape)) <= FP32_TOL


@pytest.mark.parametrize("C", [8, 16, 24, 40, 80, 7, 13])
def test_fused_channel_sweep(C):
    cache, grid, features, logits = _sweep_case(C, seed=11)
    dev = torch.device("cuda")
    fb, lb = o.bf16_round(features), o.bf16_round(logits)
    got = bp.pool_fused(torch.from_numpy(logits).to(dev).to(torch.bfloat16),
                        torch.from_numpy(features).to(dev).to(torch.bfloat16), cache, grid
                        ).values.cpu().numpy().reshape(C, -1)
    want = o.fused_pool(fb, lb, cache.ranks, cache.interval_starts, cache.interval_cells,
                        grid.n_cells, "sum")
    assert max_rel_dev(want, got) <= 1e-5


@pytest.mark.parametrize("C", [3, 32, 80])
def test_lifted_channel_sweep(C):
    cache, grid, features, logits = _sweep_case(C, seed=13)
    dist = o.normalize_depth(logits)
    dev = torch.device("cuda")
    x = bp.lift_features(torch.from_numpy(features).to(dev), torch.from_numpy(dist).to(dev))
    for red in ("sum", "mean", "max"):
        got = bp.pool_lifted(x, cache, grid, red).values.cpu().numpy().reshape(C, -1)
        want = o.pool_interval(features, dist, cache.ranks, cache.interval_starts,
                               cache.interval_cells, grid.n_cells, red)
        assert max_rel_dev(want, got) <= FP32_TOL, red


def test_fast_mode_high_res_config():
    """Config H (6 x 64 x 176, 720 x 720 grid): fast SUM within 1e-5 of the
    64-bit oracle, and the uncached builder reproduces the cached build."""
    spec = bp.CONFIGS["H"]
    rig, features, logits, grid = bp.gen_workload(spec)
    cache = bp.build_cache(rig, spec.frustum, grid)
    dist = o.normalize_depth(logits)
    want = o.pool_interval(features, dist, cache.ranks, cache.interval_starts,
                           cache.interval_cells, grid.n_cells, "sum")
    got = bp.pool_interval(features, dist, cache, grid, exact=False).values
    assert max_rel_dev(want, got.reshape(want.shape)) <= FP32_TOL
    builder = bp.CacheBuilder(spec.n_cameras, spec.frustum, grid, tiles=True)
    c2 = builder.build(torch.from_numpy(bp.rig_rows(rig)).cuda())
    got2 = bp.pool_interval(features, dist, c2, grid, exact=False).values
    assert np.array_equal(got, got2)  # per-frame tile plan (capacity-bounded), same result
    # per-frame caches without a tile plan pool with the interval kernels
    c3 = bp.CacheBuilder(spec.n_cameras, spec.frustum, grid).build(
        torch.from_numpy(bp.rig_rows(rig)).cuda())
    got3 = bp.pool_interval(features, dist, c3, grid, exact=False).values
    assert max_rel_dev(want, got3.reshape(want.shape)) <= FP32_TOL


def test_fast_mode_batched_and_deterministic():
    spec, features, logits, grid, cache = _S()
    dev = torch.device("cuda")
    F = torch.stack([torch.from_numpy(features)] * 3).to(dev)
    Dd = torch.stack([torch.from_numpy(o.normalize_depth(logits))] * 3).to(dev)
    F[1] *= -1.0
    out = bp.pool_interval(F, Dd, cache, grid, exact=False).values
    for b in range(3):
        one = bp.pool_interval(F[b], Dd[b], cache, grid, exact=False).values
        assert torch.equal(out[b], one)
    again = bp.pool_interval(F, Dd, cache, grid, exact=False).values
    assert torch.equal(out, again)


# ---- the GPU sort against a stable numpy argsort (bevgrid.py:142-158) -------
@pytest.mark.parametrize("sizes", [
    (0, 5, 31, 32, 33, 64, 65, 100, 128, 200, 256, 300, 512, 700, 1024),  # warp registers
    (1025, 3000, 8192),                 # CTA: warp-sorted slices merged by rank
    (9000, 20000),                      # in-place global fallback
])
def test_sort_intervals_every_run_length(sizes):
    """Counting-sort path (P <= 64 cells): runs of every size class, points
    shuffled and mixed with out-of-range ids, must come back in stable order."""
    rng = np.random.default_rng(len(sizes))
    n_cells = max(64, (sum(sizes) + 63) // 64 + len(sizes))
    cell_ids = rng.choice(n_cells, size=len(sizes), replace=False)
    cells = np.concatenate([np.full(n, c, dtype=np.uint32) for n, c in zip(sizes, cell_ids)]
                           + [np.full(sum(sizes) // 7 + 1, bp.OUT_OF_RANGE, dtype=np.uint32)])
    cells = cells[rng.permutation(cells.size)]
    ranks, starts, icells = bp.ranks_and_intervals(cells, n_cells)
    want = o.ranks_and_intervals(cells, n_cells)
    np.testing.assert_array_equal(ranks, want[0])
    np.testing.assert_array_equal(starts, want[1])
    np.testing.assert_array_equal(icells, want[2])


def test_sort_intervals_radix_path():
    """Few keys, long runs (P > 64 cells): the LSD radix path."""
    rng = np.random.default_rng(7)
    cells = rng.integers(0, 50, size=200_000).astype(np.uint32)
    cells[rng.random(cells.size) < 0.1] = bp.OUT_OF_RANGE
    ranks, starts, icells = bp.ranks_and_intervals(cells, 50)
    want = o.ranks_and_intervals(cells, 50)
    for got, ref in zip((ranks, starts, icells), want):
        np.testing.assert_array_equal(got, ref)


def test_per_frame_build_matches_eager():
    """A per-frame CacheBuilder build (chunk list in cell order, built beside
    the rank sort) pools like a cache built eagerly: fast within tolerance
    (the eager cache pools through the tile plan), exact bit-identical."""
    spec = bp.CONFIGS["T"]
    f = spec.frustum
    rig, feats, logits, grid = bp.gen_workload(spec)
    dist = bp.normalize_depth(logits)
    eager = bp.build_cache(rig, f, grid)
    builder = bp.CacheBuilder(spec.n_cameras, f, grid)
    lazy = builder.build(torch.from_numpy(bp.rig_rows(rig)).cuda())
    fast = bp.pool_interval(feats, dist, lazy, grid, exact=False).values
    assert max_rel_dev(bp.pool_interval(feats, dist, eager, grid, exact=True).values,
                       fast) <= FP32_TOL
    ex = bp.pool_interval(feats, dist, lazy, grid, exact=True).values
    np.testing.assert_array_equal(ex, bp.pool_interval(feats, dist, eager, grid,
                                                       exact=True).values)


def test_plan_staging_split_matches_run():
    """Interval path (MAX): PoolPlan.prepare (NHWC staging beside the zero
    fill) + reduce(zeroed) equals run(); a caller-provided output buffer is
    always zero-filled.  Tiled path (SUM): phase 1 then phase 2 equals run()."""
    spec = bp.CONFIGS["T"]
    f = spec.frustum
    rig, feats_np, logits_np, grid = bp.gen_workload(spec)
    cache = bp.build_cache(rig, f, grid)
    feats = torch.from_numpy(feats_np).cuda()[None]
    dist = bp.normalize_depth(torch.from_numpy(logits_np).cuda())[None]
    plan = bp.PoolPlan(cache, grid, spec.n_cameras, spec.channels, f.height, f.width,
                       f.depth_bins, 1, bp.Reducer.MAX)
    assert not plan.tiled
    want = plan.run(feats, dist).clone()
    plan.out.fill_(7.0)
    plan.prepare(feats)
    np.testing.assert_array_equal(plan.reduce(dist, zeroed=True).cpu().numpy(), want.cpu().numpy())
    mine = torch.full_like(want, 3.0)
    plan.reduce(dist, out=mine, zeroed=True)  # not the plan's buffer: zero-filled anyway
    np.testing.assert_array_equal(mine.cpu().numpy(), want.cpu().numpy())
    tplan = bp.PoolPlan(cache, grid, spec.n_cameras, spec.channels, f.height, f.width,
                        f.depth_bins, 1, bp.Reducer.SUM)
    assert tplan.tiled
    want = tplan.run(feats, dist).clone()
    tplan.out.fill_(7.0)
    tplan.phase(feats, dist, 1)
    np.testing.assert_array_equal(tplan.phase(feats, dist, 2).cpu().numpy(), want.cpu().numpy())


def test_run_uncached_matches_cached_pool():
    """Config-H style frame (association rebuilt beside the feature staging)
    equals pooling with an eagerly built cache."""
    spec = bp.CONFIGS["T"]
    f = spec.frustum
    rig, feats_np, logits_np, grid = bp.gen_workload(spec)
    feats = torch.from_numpy(feats_np).cuda()[None]
    dist = bp.normalize_depth(torch.from_numpy(logits_np).cuda())[None]
    builder = bp.CacheBuilder(spec.n_cameras, f, grid, tiles=True)
    cams = torch.from_numpy(bp.rig_rows(rig)).cuda()
    plan = bp.PoolPlan(builder.build(cams), grid, spec.n_cameras, spec.channels, f.height,
                       f.width, f.depth_bins, 1, bp.Reducer.SUM)
    assert plan.tiled
    got = plan.run_uncached(builder, cams, feats, dist).cpu().numpy()
    want = bp.pool_interval(feats_np, bp.normalize_depth(logits_np),
                            bp.build_cache(rig, f, grid), grid).values
    np.testing.assert_array_equal(got.reshape(want.shape), want)


@pytest.mark.parametrize("exact", [False, True])
def test_run_uncached_follows_rig_changes(exact):
    """A per-frame plan pools every frame with THAT frame's association
    (exact mode's chunk list and the tile plan included) when the rig
    changes between frames."""
    spec = bp.CONFIGS["T"]
    f = spec.frustum
    rig, feats_np, logits_np, grid = bp.gen_workload(spec)
    rig2 = [bp.CameraCalibration(c.fx * 1.1, c.fy * 1.1, c.cx + 1.5, c.cy - 0.5, c.rotation,
                                 c.translation + np.array([0.7, -0.4, 0.1]), c.camera_id)
            for c in rig]
    feats = torch.from_numpy(feats_np).cuda()[None]
    dist = bp.normalize_depth(torch.from_numpy(logits_np).cuda())[None]
    builder = bp.CacheBuilder(spec.n_cameras, f, grid)
    cams = [torch.from_numpy(bp.rig_rows(r)).cuda() for r in (rig, rig2)]
    plan = bp.PoolPlan(builder.build(cams[0]), grid, spec.n_cameras, spec.channels, f.height,
                       f.width, f.depth_bins, 1, bp.Reducer.SUM, exact=exact)
    for r, c in ((rig, cams[0]), (rig2, cams[1]), (rig, cams[0])):
        got = plan.run_uncached(builder, c, feats, dist).cpu().numpy()
        cache = bp.build_cache(r, f, grid)
        want = o.pool_interval(feats_np, dist[0].cpu().numpy(), cache.ranks,
                               cache.interval_starts, cache.interval_cells, grid.n_cells, "sum")
        if exact:
            np.testing.assert_array_equal(got.reshape(want.shape), want)
        else:
            assert max_rel_dev(want, got.reshape(want.shape)) <= FP32_TOL


@pytest.mark.parametrize("tiles", [False, True])
def test_graphed_builder_follows_rig_changes(tiles):
    """CacheBuilder(graph=True) replays one captured build per frame: its
    association arrays equal build_cache's for every rig it is fed, in any
    order, and pooling through it matches the eager builder bit for bit."""
    spec = bp.CONFIGS["S"]
    f = spec.frustum
    rig, feats_np, logits_np, grid = bp.gen_workload(spec)
    rig2 = [bp.CameraCalibration(c.fx * 0.9, c.fy * 0.9, c.cx - 2.0, c.cy + 1.0, c.rotation,
                                 c.translation + np.array([-0.3, 0.5, 0.05]), c.camera_id)
            for c in rig]
    feats = torch.from_numpy(feats_np).cuda()
    dist = bp.normalize_depth(torch.from_numpy(logits_np).cuda())
    gb = bp.CacheBuilder(spec.n_cameras, f, grid, tiles=tiles, graph=True)
    eb = bp.CacheBuilder(spec.n_cameras, f, grid, tiles=tiles)
    for r in (rig, rig2, rig2, rig):
        cams = torch.from_numpy(bp.rig_rows(r)).cuda()
        c = gb.build(cams)
        want = bp.build_cache(r, f, grid)
        for name in ("cell_of_point", "ranks", "interval_starts", "interval_cells"):
            np.testing.assert_array_equal(getattr(c, name), getattr(want, name), err_msg=name)
        got = bp.pool_interval(feats, dist, c, grid, exact=False).values
        ref = bp.pool_interval(feats, dist, eb.build(cams), grid, exact=False).values
        assert torch.equal(got, ref)


@pytest.mark.parametrize("C", [1, 3, 20, 80, 200, 250, 256, 512])
@pytest.mark.parametrize("red", ["sum", "mean", "max"])
def test_exact_mode_channel_sweep(C, red):
    """exact=True is bit-identical to the fp64 restatement for every lane
    layout: the chunk-schedule path (with its in-order walk of the long
    intervals) and, for C = 250, 512 (too wide for it), the reference-order
    kernel pool_ref.cuh."""
    cache, grid, features, logits = _sweep_case(C, seed=5)
    dist = o.normalize_depth(logits)
    want = o.pool_interval(features, dist, cache.ranks, cache.interval_starts,
                           cache.interval_cells, grid.n_cells, red)
    got = bp.pool_interval(features, dist, cache, grid, red, exact=True).values
    np.testing.assert_array_equal(got.reshape(want.shape), want)


@pytest.mark.parametrize("name", ["T", "S"])
def test_empty_cells_zeroed_beside_reduction(name):
    """PoolPlan.run replayed from a graph zeroes only the empty cells, beside
    the chunk kernel (bvp_zero_empty_cells on a forked stream); launched
    eagerly it memsets the map first.  Either way a NaN-poisoned map comes out
    equal to the oracle for every reducer, batch 2 included; the bare entry
    point zeroes exactly the cells no interval covers."""
    spec = bp.CONFIGS[name]
    f = spec.frustum
    rig, feats_np, logits_np, grid = bp.gen_workload(spec)
    cache = bp.build_cache(rig, f, grid)
    dist_np = o.normalize_depth(logits_np)
    feats = torch.from_numpy(np.stack([feats_np, -feats_np])).cuda()
    dist = torch.from_numpy(np.stack([dist_np, dist_np])).cuda()
    for red in bp.Reducer:
        plan = bp.PoolPlan(cache, grid, spec.n_cameras, spec.channels, f.height, f.width,
                           f.depth_bins, 2, red)
        g = plan.graphed(plan.run, feats, dist)  # captured: zero fill beside the kernels
        for run in (lambda: plan.run(feats, dist), g.replay):  # eager: memset first
            plan.out.fill_(float("nan"))
            run()
            got = plan.out.cpu().numpy()
            for b, fb in enumerate((feats_np, -feats_np)):
                want = o.pool_interval(fb, dist_np, cache.ranks, cache.interval_starts,
                                       cache.interval_cells, grid.n_cells, red.value)
                assert max_rel_dev(want, got[b].reshape(want.shape)) <= FP32_TOL, (red, b)
    out = torch.full((2, spec.channels, grid.n_cells), float("nan"), device="cuda")
    bp._lib.call("bvp_zero_empty_cells", cache.d_cell_first.data_ptr(), grid.n_cells,
                 spec.channels, 2, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    occupied = np.zeros(grid.n_cells, bool)
    occupied[np.asarray(cache.interval_cells)] = True
    o_np = out.cpu().numpy()
    assert np.isnan(o_np[:, :, occupied]).all()
    assert (o_np[:, :, ~occupied] == 0).all()


# ---- the fused path's backward (config F training) vs the fp64 restatement ----

def _fused_grads(name, red, seed=3):
    spec = bp.CONFIGS[name]
    rig, features, logits, grid = bp.gen_workload(spec)
    cache = bp.build_cache(rig, spec.frustum, grid)
    dev = torch.device("cuda")
    lg = torch.from_numpy(logits).to(dev).to(torch.bfloat16).requires_grad_(True)
    cx = torch.from_numpy(features).to(dev).to(torch.bfloat16).requires_grad_(True)
    out = bp.bev_pool_fused(lg, cx, cache, grid, red)
    g = torch.randn(out.shape, device=dev, generator=torch.Generator(dev).manual_seed(seed))
    out.backward(g)
    assert lg.grad.dtype == torch.bfloat16 and cx.grad.dtype == torch.bfloat16
    return (spec, features, logits, grid, cache, out.detach(), g.cpu().numpy().reshape(out.shape[0], -1),
            lg.grad.float().cpu().numpy(), cx.grad.float().cpu().numpy())


@pytest.mark.parametrize("red", ["sum", "mean"])
def test_fused_backward_matches_fp64_restatement(red):
    spec, features, logits, grid, cache, out, g, gl, gc = _fused_grads("T", red)
    want_l, want_c = o.fused_backward(o.bf16_round(features), o.bf16_round(logits),
                                      cache.cell_of_point, g, cache.ranks,
                                      cache.interval_starts, cache.interval_cells, red)
    assert max_rel_dev(want_l, gl) <= BF16_TOL
    assert max_rel_dev(want_c, gc) <= BF16_TOL
    want = o.fused_pool(o.bf16_round(features), o.bf16_round(logits), cache.ranks,
                        cache.interval_starts, cache.interval_cells, grid.n_cells, red)
    assert max_rel_dev(want, out.cpu().numpy().reshape(want.shape)) <= 1e-5


def test_fused_backward_nuscenes_shape_sum():
    """S shape, restated per camera in fp64 (as test_backward_nuscenes_shape_sum)."""
    spec, features, logits, grid, cache, out, g, gl_got, gc_got = _fused_grads("S", "sum")
    fb, lb = o.bf16_round(features).astype(np.float64), o.bf16_round(logits).astype(np.float64)
    N, C, H, W = features.shape
    D = logits.shape[1]
    cells = cache.cell_of_point.reshape(N, H, W, D)
    g64 = np.concatenate([g.astype(np.float64), np.zeros((C, 1))], axis=1)
    for n in range(N):
        e = np.exp(lb[n] - lb[n].max(axis=0, keepdims=True))
        w = e / e.sum(axis=0, keepdims=True)                      # D, H, W
        idx = np.where(cells[n] == bp.OUT_OF_RANGE, grid.n_cells, cells[n]).astype(np.int64)
        gcol = g64[:, idx]                                        # C, H, W, D
        gc = np.einsum("chwd,dhw->chw", gcol, w)
        gw = np.einsum("chwd,chw->dhw", gcol, fb[n])
        gl = w * (gw - (w * gw).sum(axis=0, keepdims=True))
        assert max_rel_dev(gc, gc_got[n]) <= BF16_TOL
        assert max_rel_dev(gl, gl_got[n]) <= BF16_TOL


@pytest.mark.parametrize("name", ["T", "S", "H"])
def test_tile_plan_from_ranks_matches_per_tile_sort(name):
    """bvp_build_tile_plan_ranks (the association's ranks stably sorted by
    tile) and bvp_build_tile_plan (a bitonic sort per tile) build the same
    plan: same segment count, and the tiled reduction through either is bit
    for bit the same map (SUM and MEAN, fp32 and the fused bf16 variant)."""
    from paper_2205_13542_b200.bevgrid import TilePlan
    spec = bp.CONFIGS[name]
    f = spec.frustum
    rig, feats_np, logits_np, grid = bp.gen_workload(spec)
    cache = bp.build_cache(rig, f, grid)
    dims = (spec.n_cameras, f.height, f.width, f.depth_bins)
    dev = torch.device("cuda")
    a = TilePlan(*dims, grid.n_cells, dev).build(cache.d_cell_of_point, exact_count=True)
    b = TilePlan(*dims, grid.n_cells, dev).build(cache.d_cell_of_point, exact_count=True,
                                                 ranks=cache.d_ranks, counts=cache.d_counts)
    assert a.n_seg == b.n_seg
    feats = torch.from_numpy(feats_np).to(dev)
    dist = bp.normalize_depth(torch.from_numpy(logits_np).to(dev))
    C = spec.channels
    for mode in (bp._lib.BVP_SUM, bp._lib.BVP_MEAN):
        oa = torch.empty(C * grid.n_cells, device=dev)
        ob = torch.empty(C * grid.n_cells, device=dev)
        a.pool_f32(feats, dist, 1, C, mode, oa)
        b.pool_f32(feats, dist, 1, C, mode, ob)
        assert torch.equal(oa, ob)
    lg = torch.from_numpy(logits_np).to(dev).to(torch.bfloat16)
    cx = feats.to(torch.bfloat16)
    oa = torch.empty(C * grid.n_cells, device=dev)
    ob = torch.empty(C * grid.n_cells, device=dev)
    a.pool_fused_bf16(lg, cx, 1, C, bp._lib.BVP_SUM, oa)
    b.pool_fused_bf16(lg, cx, 1, C, bp._lib.BVP_SUM, ob)
    assert torch.equal(oa, ob)


@pytest.mark.parametrize("seed", [20_000 + s for s in range(8)])
def test_tile_path_random_wide_instances(seed):
    """Random rigs with up to 96 rows (several 64-row tiles per column), up to
    130 depth bins (depth-weight quads past 32) and odd widths (clusters of
    8 / 4 / 2 / 1 columns): the tiled reduction (SUM, MEAN) and its fused
    bf16 variant against the 64-bit oracle."""
    inst = random_instance(seed, 96, 130, 40)
    frustum, grid = specs_of(inst)
    cache = bp.build_cache(rig_of(inst.cams), frustum, grid)
    dist = o.normalize_depth(inst.logits)
    C = inst.features.shape[1]
    n_cam = inst.cams.shape[0]
    assert cache.tile_plan(n_cam, frustum.height, frustum.width, frustum.depth_bins) is not None
    for red in (bp.Reducer.SUM, bp.Reducer.MEAN):
        want = o.pool_naive(inst.features, dist, cache.cell_of_point, grid.n_cells, red.value)
        got = bp.pool_interval(inst.features, dist, cache, grid, red, exact=False)
        assert max_rel_dev(want, got.values.reshape(want.shape)) <= FP32_TOL, red
    if C == 0:
        return
    dev = torch.device("cuda")
    fb, lb = o.bf16_round(inst.features), o.bf16_round(inst.logits)
    got = bp.pool_fused(torch.from_numpy(inst.logits).to(dev).to(torch.bfloat16),
                        torch.from_numpy(inst.features).to(dev).to(torch.bfloat16), cache, grid
                        ).values.cpu().numpy().reshape(C, -1)
    want = o.fused_pool(fb, lb, cache.ranks, cache.interval_starts, cache.interval_cells,
                        grid.n_cells, "sum")
    assert max_rel_dev(want, got) <= 1e-5


@pytest.mark.parametrize("seed", [20_000 + s for s in range(6)])
@pytest.mark.parametrize("red", ["sum", "mean"])
def test_tiled_backward_random_wide_instances(seed, red):
    """bev_pool's SUM / MEAN backward (tiled forward, gather backward) and the
    tiled adjoint (bvp_tile_backward_f32) on random wide rigs against the
    fp64 restatement: gradients of both the features and the depth
    distribution, out-of-range points and pixels without in-range points
    included (zeros)."""
    inst = random_instance(seed, 96, 130, 40)
    frustum, grid = specs_of(inst)
    cache = bp.build_cache(rig_of(inst.cams), frustum, grid)
    dist = o.normalize_depth(inst.logits)
    C = inst.features.shape[1]
    if C == 0:
        return
    dev = torch.device("cuda")
    f = torch.from_numpy(inst.features).to(dev).requires_grad_(True)
    d = torch.from_numpy(dist).to(dev).requires_grad_(True)
    out = bp.bev_pool(f, d, cache, grid, red)
    g = np.random.default_rng(seed).standard_normal((C, grid.n_cells)).astype(np.float32)
    out.backward(torch.from_numpy(g).to(dev).view_as(out))
    gf, gw = o.pool_backward(inst.features, dist, cache.cell_of_point, g.astype(np.float64),
                             cache.ranks, cache.interval_starts, cache.interval_cells, red)
    assert max_rel_dev(gf, f.grad.cpu().numpy()) <= FP32_TOL
    assert max_rel_dev(gw, d.grad.cpu().numpy()) <= FP32_TOL
    n_cam = inst.cams.shape[0]
    tp = cache.tile_plan(n_cam, frustum.height, frustum.width, frustum.depth_bins)
    tf = torch.full_like(f, float("nan"))
    tw = torch.full_like(d, float("nan"))
    tp.backward_f32(torch.from_numpy(g).to(dev), f.detach(), d.detach(), 1, C,
                    bp._lib.BVP_MEAN if red == "mean" else bp._lib.BVP_SUM, tf, tw)
    assert max_rel_dev(gf, tf.cpu().numpy()) <= FP32_TOL
    assert max_rel_dev(gw, tw.cpu().numpy()) <= FP32_TOL
    # either gradient alone: the same bits (deterministic, independent parts)
    tw2 = torch.full_like(d, float("nan"))
    tp.backward_f32(torch.from_numpy(g).to(dev), f.detach(), d.detach(), 1, C,
                    bp._lib.BVP_MEAN if red == "mean" else bp._lib.BVP_SUM, None, tw2)
    assert torch.equal(tw, tw2)
    tf2 = torch.full_like(f, float("nan"))
    tp.backward_f32(torch.from_numpy(g).to(dev), f.detach(), d.detach(), 1, C,
                    bp._lib.BVP_MEAN if red == "mean" else bp._lib.BVP_SUM, tf2, None)
    assert torch.equal(tf, tf2)


def test_tiled_adjoints_zero_channels():
    """C = 0: the map is empty, so both adjoints write an all-zero weight /
    logit gradient (and touch nothing else)."""
    spec = bp.CONFIGS["T"]
    f = spec.frustum
    rig, _, logits, grid = bp.gen_workload(spec)
    cache = bp.build_cache(rig, f, grid)
    tp = cache.tile_plan(spec.n_cameras, f.height, f.width, f.depth_bins)
    dev = torch.device("cuda")
    N, D, H, W = logits.shape
    g = torch.empty((1, 0, grid.n_cells), device=dev)
    feats = torch.empty((1, N, 0, H, W), device=dev)
    dist = torch.from_numpy(o.normalize_depth(logits)).to(dev)[None]
    gw = torch.full_like(dist, float("nan"))
    tp.backward_f32(g, feats, dist, 1, 0, bp._lib.BVP_SUM, None, gw)
    assert (gw == 0).all()
    lg = torch.from_numpy(logits).to(dev).to(torch.bfloat16)[None]
    gl = torch.full_like(lg, float("nan"))
    tp.fused_backward_bf16(g, lg, feats.to(torch.bfloat16), 1, 0, bp._lib.BVP_SUM, gl, None)
    assert (gl == 0).all()


@pytest.mark.parametrize("seed", [21_000 + s for s in range(6)])
@pytest.mark.parametrize("red", ["sum", "mean"])
def test_tiled_fused_backward_random_instances(seed, red):
    """bev_pool_fused's backward (bvp_tile_fused_backward_bf16: the softmax
    re-formed per tile, bf16 gradients out) on random rigs against the fp64
    restatement, and against the two-pass fallback (bvp_fused_backward_bf16:
    fp32 softmax + gather backward + Jacobian kernel); either gradient alone
    gives the same bits."""
    inst = random_instance(seed, 96, 130, 40)
    frustum, grid = specs_of(inst)
    cache = bp.build_cache(rig_of(inst.cams), frustum, grid)
    C = inst.features.shape[1]
    if C == 0:
        return
    dev = torch.device("cuda")
    lg = torch.from_numpy(inst.logits).to(dev).to(torch.bfloat16).requires_grad_(True)
    cx = torch.from_numpy(inst.features).to(dev).to(torch.bfloat16).requires_grad_(True)
    out = bp.bev_pool_fused(lg, cx, cache, grid, red)
    g = np.random.default_rng(seed).standard_normal((C, grid.n_cells)).astype(np.float32)
    out.backward(torch.from_numpy(g).to(dev).view_as(out))
    want_l, want_c = o.fused_backward(o.bf16_round(inst.features), o.bf16_round(inst.logits),
                                      cache.cell_of_point, g.astype(np.float64), cache.ranks,
                                      cache.interval_starts, cache.interval_cells, red)
    assert max_rel_dev(want_l, lg.grad.float().cpu().numpy()) <= BF16_TOL
    assert max_rel_dev(want_c, cx.grad.float().cpu().numpy()) <= BF16_TOL
    N, D, H, W = inst.logits.shape
    mode = bp._lib.BVP_MEAN if red == "mean" else bp._lib.BVP_SUM
    gd = torch.from_numpy(g).to(dev)[None]
    l5, c5 = lg.detach()[None].contiguous(), cx.detach()[None].contiguous()
    ws = torch.empty(int(bp._lib.load().bvp_fused_backward_workspace_bytes(
        1, N, C, H, W, D, cache.n_int_max)), dtype=torch.uint8, device=dev)
    fl, fc = torch.empty_like(l5), torch.empty_like(c5)
    bp._lib.call("bvp_fused_backward_bf16", gd.data_ptr(), l5.data_ptr(), c5.data_ptr(),
                 cache.d_interval_starts.data_ptr(), cache.d_interval_cells.data_ptr(),
                 cache.d_cell_first.data_ptr(), cache.d_interval_of_point.data_ptr(), 1, N, C,
                 H, W, D, grid.nx, grid.ny, cache.n_int_max, mode, fl.data_ptr(),
                 fc.data_ptr(), ws.data_ptr(), ws.numel(),
                 torch.cuda.current_stream().cuda_stream)
    assert max_rel_dev(want_l, fl[0].float().cpu().numpy()) <= BF16_TOL
    assert max_rel_dev(want_c, fc[0].float().cpu().numpy()) <= BF16_TOL
    tp = cache.tile_plan(N, H, W, D)
    tl2 = torch.full_like(l5, float("nan"))
    tp.fused_backward_bf16(gd, l5, c5, 1, C, mode, tl2, None)
    assert torch.equal(tl2[0], lg.grad)
    tc2 = torch.full_like(c5, float("nan"))
    tp.fused_backward_bf16(gd, l5, c5, 1, C, mode, None, tc2)
    assert torch.equal(tc2[0], cx.grad)


@pytest.mark.parametrize("seed", [30_000 + s for s in range(4)])
def test_tile_path_random_deep_instances(seed):
    """Up to 600 depth bins (tiles of fewer rows, several rounds of depth
    quads per CTA, the fused softmax over long rays): the tiled reduction
    and its fused variant against the 64-bit oracle."""
    inst = random_instance(seed, 24, 600, 12)
    frustum, grid = specs_of(inst)
    cache = bp.build_cache(rig_of(inst.cams), frustum, grid)
    dist = o.normalize_depth(inst.logits)
    C = inst.features.shape[1]
    for red in (bp.Reducer.SUM, bp.Reducer.MEAN):
        want = o.pool_naive(inst.features, dist, cache.cell_of_point, grid.n_cells, red.value)
        got = bp.pool_interval(inst.features, dist, cache, grid, red, exact=False)
        assert max_rel_dev(want, got.values.reshape(want.shape)) <= FP32_TOL, red
    if C == 0:
        return
    dev = torch.device("cuda")
    fb, lb = o.bf16_round(inst.features), o.bf16_round(inst.logits)
    got = bp.pool_fused(torch.from_numpy(inst.logits).to(dev).to(torch.bfloat16),
                        torch.from_numpy(inst.features).to(dev).to(torch.bfloat16), cache, grid
                        ).values.cpu().numpy().reshape(C, -1)
    want = o.fused_pool(fb, lb, cache.ranks, cache.interval_starts, cache.interval_cells,
                        grid.n_cells, "sum")
    assert max_rel_dev(want, got) <= 1e-5
