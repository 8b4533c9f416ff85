"""Batch sharding on CPU: world_size-2 gloo process groups.

The GPU path shards whole samples over ranks with no data-path collective;
these tests pin the host logic -- the sample partition, the seeds, the
max-over-ranks timing reduction and the gather of per-rank BEV maps to rank
0 -- with the oracle standing in for the per-rank pooling (tests only).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

from oracle import oracle as o
from paper_2205_13542_b200.shard import (
    gather_maps,
    max_over_ranks,
    sample_seeds,
    shard_range,
    sum_over_ranks,
)


@pytest.mark.parametrize("n,world", [(0, 1), (1, 1), (4, 2), (8, 8), (5, 2), (3, 4), (9, 4)])
def test_shard_range_partitions(n, world):
    seen = []
    sizes = []
    for r in range(world):
        lo, hi = shard_range(n, r, world)
        assert 0 <= lo <= hi <= n
        seen.extend(range(lo, hi))
        sizes.append(hi - lo)
    assert seen == list(range(n))
    assert max(sizes) - min(sizes) <= 1


def test_shard_range_rejects_bad_rank():
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)
    with pytest.raises(ValueError):
        shard_range(-1, 0, 1)


def test_sample_seeds_are_sample_indices():
    assert sample_seeds(8, 3, 4) == [6, 7]
    assert sample_seeds(4, 0, 1, base_seed=10) == [10, 11, 12, 13]


def _pool_sample(seed: int, cache) -> np.ndarray:
    cfg = o.CONFIGS["T"]
    f, lg = o.gen_inputs(cfg.n_cameras, cfg.channels, cfg.height, cfg.width, cfg.depth_bins, seed)
    return o.pool_interval(f, o.normalize_depth(lg), cache["ranks"], cache["interval_starts"],
                           cache["interval_cells"], cfg.n_cells, "sum")


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _pool_sample_cuda(seed: int) -> np.ndarray:
    """The same sample pooled by the CUDA path (exact mode: the reference's
    bits, so the oracle's single-process result must match exactly)."""
    import paper_2205_13542_b200 as bp
    spec = bp.CONFIGS["T"]
    rig, f, lg, grid = bp.gen_workload(bp.WorkloadSpec(spec.n_cameras, spec.frustum, spec.grid,
                                                       spec.channels, seed))
    cache = bp.build_cache(rig, spec.frustum, grid)
    return bp.pool_interval(f, o.normalize_depth(lg), cache, grid, exact=True).values


def _worker(rank: int, world: int, port: int, n_samples: int, out_path: str,
            cuda: bool = False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = o.CONFIGS["T"]
        cache = o.build_cache(cfg)  # deterministic: identical on every rank
        seeds = sample_seeds(n_samples, rank, world)
        local = ([_pool_sample_cuda(s) for s in seeds] if cuda else
                 [_pool_sample(s, cache) for s in seeds])
        block = torch.from_numpy(np.stack(local)).reshape(len(local), cfg.channels, cfg.nx, cfg.ny)
        full = gather_maps(block, n_samples)
        t_max = max_over_ranks(1.0 + rank)
        t_sum = sum_over_ranks(1.0)
        if rank == 0:
            np.save(out_path, full.numpy())
            assert t_max == float(world)
            assert t_sum == float(world)
        else:
            assert full is None
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("n_samples", [4, 3])
def test_two_rank_gather_matches_single_process(tmp_path, n_samples):
    out_path = str(tmp_path / "full.npy")
    mp.spawn(_worker, args=(2, _free_port(), n_samples, out_path), nprocs=2, join=True)
    full = np.load(out_path)
    cfg = o.CONFIGS["T"]
    cache = o.build_cache(cfg)
    want = np.stack([_pool_sample(s, cache) for s in range(n_samples)])
    assert full.shape == (n_samples, cfg.channels, cfg.nx, cfg.ny)
    assert np.array_equal(full.reshape(want.shape), want)  # bit-identical: shards are independent


@pytest.mark.gpu
def test_two_rank_cuda_pooling_gather_matches_single_process(tmp_path):
    """Both ranks pool through the CUDA path (sharing the one GPU), gloo
    gathers the maps: bit-identical to the single-process oracle."""
    out_path = str(tmp_path / "full.npy")
    mp.spawn(_worker, args=(2, _free_port(), 4, out_path, True), nprocs=2, join=True)
    full = np.load(out_path)
    cfg = o.CONFIGS["T"]
    cache = o.build_cache(cfg)
    want = np.stack([_pool_sample(s, cache) for s in range(4)])
    assert np.array_equal(full.reshape(want.shape), want)


def test_single_process_helpers_are_identity():
    t = torch.arange(6.0).reshape(1, 1, 2, 3)
    assert gather_maps(t, 1) is t
    assert max_over_ranks(3.5) == 3.5
    assert sum_over_ranks(2.0) == 2.0
