"""Batch sharding over ranks: one process per GPU, whole
samples per rank, no collective on the data path.

The reference has no batch API and no distributed backend (every entry point
takes one rig / one sample, pooling.py:206-240); samples are independent, so
the B200 build shards them: rank g pools samples [lo_g, hi_g) with its own
copy of the (deterministic, identical) association cache.  torch.distributed
-- NCCL on the GPU box, gloo in the CPU tests -- is used only to
  * reduce per-rank timings to the max over ranks (bench.py), and
  * gather per-rank BEV maps / checksums to rank 0 for verification,
both outside any timed region.
"""

from __future__ import annotations

import torch
import torch.distributed as tdist


def shard_range(n_samples: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of samples for ``rank``: sizes differ by at most one,
    lower ranks take the remainder, every sample is owned exactly once."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    if n_samples < 0:
        raise ValueError(f"bad sample count {n_samples}")
    base, extra = divmod(n_samples, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def sample_seeds(n_samples: int, rank: int, world: int, base_seed: int = 0) -> list[int]:
    """Seeds of this rank's samples: sample b uses seed base_seed + b
    (batch sample b uses seed b)."""
    lo, hi = shard_range(n_samples, rank, world)
    return [base_seed + b for b in range(lo, hi)]


def _initialized() -> bool:
    return tdist.is_available() and tdist.is_initialized()


def _coll_device(device):
    """gloo reduces host tensors; NCCL device tensors."""
    return None if tdist.get_backend() == "gloo" else device


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device-timed step time) over all ranks."""
    if not _initialized() or tdist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_coll_device(device))
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    return float(t.item())


def gather_scalars(value: float, device=None) -> list[float]:
    """Every rank's scalar (e.g. its device-timed step), in rank order."""
    if not _initialized() or tdist.get_world_size() == 1:
        return [float(value)]
    t = torch.tensor([float(value)], dtype=torch.float64, device=_coll_device(device))
    bufs = [torch.empty_like(t) for _ in range(tdist.get_world_size())]
    tdist.all_gather(bufs, t)
    return [float(b.item()) for b in bufs]


def sum_over_ranks(value: float, device=None) -> float:
    if not _initialized() or tdist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_coll_device(device))
    tdist.all_reduce(t, op=tdist.ReduceOp.SUM)
    return float(t.item())


def gather_maps(local: torch.Tensor, n_samples: int) -> torch.Tensor | None:
    """Gather every rank's (b_local, C, nx, ny) block of BEV maps to rank 0 as
    one (n_samples, C, nx, ny) tensor in sample order; other ranks get None.
    Uneven shards are padded to the largest block for the collective."""
    if not _initialized() or tdist.get_world_size() == 1:
        return local
    world, rank = tdist.get_world_size(), tdist.get_rank()
    if tdist.get_backend() == "gloo":
        local = local.cpu()  # gloo gathers host tensors
    sizes = [shard_range(n_samples, r, world) for r in range(world)]
    cap = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((cap, *local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    tdist.all_gather(bufs, pad)
    if rank != 0:
        return None
    return torch.cat([bufs[r][: hi - lo] for r, (lo, hi) in enumerate(sizes)])
