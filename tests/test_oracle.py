"""The CPU oracle, pinned bit-for-bit to digests of the reference's own
outputs (tests/golden/golden.json, produced by tests/golden/make_golden.py
importing the reference).  CPU only."""

import numpy as np
import pytest

from conftest import max_rel_dev, sha
from instances import GOLDEN_INSTANCES, random_instance
from oracle import oracle as o


def _check(entry, cams, h, w, d, dmin, dstep, grid, nx, ny, features, logits):
    cells = o.frustum_cells(cams, h, w, d, dmin, dstep, grid, nx, ny)
    ranks, starts, icells = o.ranks_and_intervals(cells, nx * ny)
    dist = o.normalize_depth(logits)
    assert ranks.size == entry["n_in"] and starts.size == entry["n_int"]
    got = {"cell_of_point": sha(cells), "ranks": sha(ranks), "interval_starts": sha(starts),
           "interval_cells": sha(icells), "dist": sha(dist)}
    for m in ("sum", "mean", "max"):
        got["pool_" + m] = sha(o.pool_interval(features, dist, ranks, starts, icells, nx * ny, m))
    bad = [k for k, v in got.items() if entry["sha256"][k] != v]
    assert not bad, f"oracle differs from the reference on {bad}"


@pytest.mark.parametrize("name", ["T", "S", "H"])
def test_oracle_matches_reference_configs(golden, name):
    cfg = o.CONFIGS[name]
    cams = o.synthetic_rig(cfg.n_cameras, cfg.height, cfg.width)
    f, lg = o.gen_inputs(cfg.n_cameras, cfg.channels, cfg.height, cfg.width, cfg.depth_bins, 0)
    entry = golden["configs"][name]
    assert sha(f) == entry["sha256"]["features"] and sha(lg) == entry["sha256"]["logits"]
    _check(entry, cams, cfg.height, cfg.width, cfg.depth_bins, cfg.depth_min, cfg.depth_step,
           cfg.grid, cfg.nx, cfg.ny, f, lg)


@pytest.mark.parametrize("seed,mhw,md,mc", GOLDEN_INSTANCES)
def test_oracle_matches_reference_instances(golden, seed, mhw, md, mc):
    i = random_instance(seed, mhw, md, mc)
    _check(golden["instances"][str(seed)], i.cams, i.height, i.width, i.depth_bins, i.depth_min,
           i.depth_step, i.grid, i.nx, i.ny, i.features, i.logits)


def test_oracle_T_arrays_match_stored_golden():
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_T.npz"))
    c = o.build_cache(o.CONFIGS["T"])
    for k in ("cell_of_point", "ranks", "interval_starts", "interval_cells"):
        np.testing.assert_array_equal(c[k], g[k])


# ---- reference KATs restated on the oracle (test_bevgrid.py:77-108,
# test_pooling.py:141-183 of the reference suite) ----------------------------

def test_ranks_worked_example():
    ranks, starts, cells = o.ranks_and_intervals(np.array([2, 0, 2, 1], np.uint32), 3)
    np.testing.assert_array_equal(ranks, [1, 3, 0, 2])
    np.testing.assert_array_equal(starts, [0, 1, 2])
    np.testing.assert_array_equal(cells, [0, 1, 2])


def test_ranks_all_out_of_range():
    r, s, c = o.ranks_and_intervals(np.full(10, o.OUT_OF_RANGE, np.uint32), 4)
    assert r.size == s.size == c.size == 0


def _worked():
    features = np.array([1, 2, 3, 4], np.float32).reshape(1, 1, 1, 4)
    dist = np.ones((1, 1, 1, 4), np.float32)
    cells = np.array([2, 0, 2, 1], np.uint32)
    return features, dist, cells


@pytest.mark.parametrize("mode,want", [("sum", [2, 4, 4]), ("mean", [2, 4, 2]), ("max", [2, 4, 3])])
def test_pool_worked_example(mode, want):
    f, d, cells = _worked()
    r, s, c = o.ranks_and_intervals(cells, 3)
    np.testing.assert_array_equal(o.pool_interval(f, d, r, s, c, 3, mode).reshape(3), want)
    np.testing.assert_array_equal(o.pool_naive(f, d, cells, 3, mode).reshape(3), want)


def test_prefixsum_by_hand():
    f, d, cells = _worked()
    r, s, c = o.ranks_and_intervals(cells, 3)
    np.testing.assert_array_equal(f.reshape(-1)[r], [2, 4, 1, 3])
    np.testing.assert_array_equal(o.prefixsum_pool(f, d, r, s, c, 3).reshape(3), [2, 4, 4])


@pytest.mark.parametrize("seed", [100, 101, 102, 10_000])
def test_naive_prefixsum_interval_agree(seed):
    i = random_instance(seed)
    cells = o.frustum_cells(i.cams, i.height, i.width, i.depth_bins, i.depth_min, i.depth_step,
                            i.grid, i.nx, i.ny)
    r, s, c = o.ranks_and_intervals(cells, i.n_cells)
    dist = o.normalize_depth(i.logits)
    for m in ("sum", "mean", "max"):
        a = o.pool_naive(i.features, dist, cells, i.n_cells, m)
        b = o.pool_interval(i.features, dist, r, s, c, i.n_cells, m)
        assert max_rel_dev(a, b) < 1e-6
        if m != "max":
            assert max_rel_dev(a, o.prefixsum_pool(i.features, dist, r, s, c, i.n_cells, m)) < 1e-4


def test_backward_oracle_finite_differences():
    """The fp64 backward restatement against central differences."""
    i = random_instance(6, max_hw=6, max_d=4, max_c=3)  # 96 points, C=3
    cells = o.frustum_cells(i.cams, i.height, i.width, i.depth_bins, i.depth_min, i.depth_step,
                            i.grid, i.nx, i.ny)
    r, s, c = o.ranks_and_intervals(cells, i.n_cells)
    if r.size == 0 or i.features.shape[1] == 0:
        pytest.skip("degenerate instance")
    dist = o.normalize_depth(i.logits)
    rng = np.random.default_rng(0)
    g = rng.normal(size=(i.features.shape[1], i.n_cells))

    def loss(f, w, mode):
        ff = f.astype(np.float64)
        ww = w.astype(np.float64)
        N, C, H, W = ff.shape
        D = ww.shape[1]
        out = np.zeros((C, i.n_cells))
        bounds = np.append(s.astype(np.int64), r.size)
        for k in range(s.size):
            pts = r[bounds[k]:bounds[k + 1]].astype(np.int64)
            d_ = pts % D
            rest = pts // D
            w_ = rest % W
            rest //= W
            h_ = rest % H
            n_ = rest // H
            vals = ww[n_, d_, h_, w_][:, None] * ff[n_, :, h_, w_]
            out[:, c[k]] = {"sum": vals.sum(0), "mean": vals.mean(0), "max": vals.max(0)}[mode]
        return float((out * g).sum())

    for mode in ("sum", "mean", "max"):
        gf, gw = o.pool_backward(i.features, dist, cells, g, r, s, c, mode)
        eps = 1e-6
        for arr, grad in ((i.features, gf), (dist, gw)):
            flat = arr.reshape(-1)
            for idx in rng.choice(flat.size, size=min(6, flat.size), replace=False):
                a = arr.astype(np.float64)
                fa = a.reshape(-1)
                fa[idx] += eps
                up = loss(a if arr is i.features else i.features, dist if arr is i.features else a, mode)
                fa[idx] -= 2 * eps
                dn = loss(a if arr is i.features else i.features, dist if arr is i.features else a, mode)
                num = (up - dn) / (2 * eps)
                assert abs(num - grad.reshape(-1)[idx]) < 1e-5 * max(1.0, abs(num)), (mode, idx)
