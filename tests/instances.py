"""Seeded test instances, restating the reference suite's generators.

``random_instance`` restates the reference's tests/conftest.py:13-65
(random_rotation, random_calibration, random_grid, random_instance) call for
call on the same numpy Generator, so seed k here yields exactly the inputs the
reference's own tests use for seed k.  Cameras are returned as the (N, 16)
float64 rows fx, fy, cx, cy, R[9], t[3] used by the C-ABI and the oracle.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Instance:
    cams: np.ndarray          # (N, 16) float64
    height: int
    width: int
    depth_bins: int
    depth_min: float
    depth_step: float
    grid: tuple               # x_min, x_max, y_min, y_max, z_min, z_max, r
    nx: int
    ny: int
    features: np.ndarray      # (N, C, H, W) float32
    logits: np.ndarray        # (N, D, H, W) float32

    @property
    def n_cells(self):
        return self.nx * self.ny

    @property
    def n_cameras(self):
        return self.cams.shape[0]


def _random_rotation(rng):
    q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


def _random_calibration(rng):
    fx = float(rng.uniform(20.0, 120.0))
    fy = float(rng.uniform(20.0, 120.0))
    cx = float(rng.uniform(5.0, 50.0))
    cy = float(rng.uniform(5.0, 50.0))
    rot = _random_rotation(rng)
    t = rng.uniform(-3.0, 3.0, size=3)
    return np.concatenate([[fx, fy, cx, cy], rot.reshape(-1), t])


def _random_grid(rng):
    r = float(rng.choice([0.25, 0.4, 0.5, 1.0]))
    nx = int(rng.integers(4, 48))
    ny = int(rng.integers(4, 48))
    x_min = float(rng.integers(-20, 4)) * r
    y_min = float(rng.integers(-20, 4)) * r
    grid = (x_min, x_min + nx * r, y_min, y_min + ny * r, -5.0, 8.0, r)
    # BevGridSpec.nx = round((x_max - x_min) / r)  (bevgrid.py:58-64)
    return grid, int(round((grid[1] - grid[0]) / r)), int(round((grid[3] - grid[2]) / r))


def random_instance(seed: int, max_hw: int = 24, max_d: int = 12, max_c: int = 8) -> Instance:
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 7))
    h = int(rng.integers(1, max_hw + 1))
    w = int(rng.integers(1, max_hw + 1))
    d = int(rng.integers(1, max_d + 1))
    c = int(rng.integers(0, max_c + 1))
    dmin = float(rng.uniform(0.5, 2.0))
    dstep = float(rng.uniform(0.25, 1.0))
    cams = np.array([_random_calibration(rng) for _ in range(n)], dtype=np.float64)
    grid, nx, ny = _random_grid(rng)
    features = rng.uniform(-1, 1, size=(n, c, h, w)).astype(np.float32)
    logits = rng.uniform(-3, 3, size=(n, d, h, w)).astype(np.float32)
    return Instance(cams, h, w, d, dmin, dstep, grid, nx, ny, features, logits)


#: seeds and size caps of the instances pinned in tests/golden/golden.json
#: (reference seeds: test_pooling.py:185-215 uses 0-7, 100-111, 300-305;
#: test_acceptance.py:64-89 uses 10_000+ with max_hw=64, max_d=32, max_c=16)
GOLDEN_INSTANCES = (
    [(s, 24, 12, 8) for s in (0, 1, 2, 3, 17, 21, 33, 40)]
    + [(100 + s, 24, 12, 8) for s in range(12)]
    + [(300 + s, 24, 12, 8) for s in range(6)]
    + [(10_000 + s, 64, 32, 16) for s in range(12)]
)


# ---- shared-BEV fusion inputs (tests/golden/make_golden_fusion.py) ---------

def random_cloud(seed: int, n: int, grid: tuple) -> np.ndarray:
    """(n, 4) float64 LiDAR-like cloud over and around `grid`: a quarter of
    the x/y coordinates sit exactly on cell edges, some points fall outside
    x/y/z, intensities in [0, 1)."""
    rng = np.random.default_rng(seed)
    x_min, x_max, y_min, y_max, z_min, z_max, r = grid
    pts = np.empty((n, 4))
    pts[:, 0] = rng.uniform(x_min - 2 * r, x_max + 2 * r, n)
    pts[:, 1] = rng.uniform(y_min - 2 * r, y_max + 2 * r, n)
    edge = rng.random(n) < 0.25
    pts[edge, 0] = x_min + r * rng.integers(-1, int(round((x_max - x_min) / r)) + 2, edge.sum())
    pts[edge, 1] = y_min + r * rng.integers(-1, int(round((y_max - y_min) / r)) + 2, edge.sum())
    pts[:, 2] = rng.uniform(z_min - 1.0, z_max + 1.0, n)
    pts[:, 3] = rng.random(n)
    return pts


#: (seed, points, grid) of the pinned LiDAR cases
LIDAR_CASES = [
    (1, 20000, (-51.2, 51.2, -51.2, 51.2, -10.0, 10.0, 0.8)),
    (2, 100000, (-54.0, 54.0, -54.0, 54.0, -10.0, 10.0, 0.3)),
    (3, 0, (-8.0, 8.0, -8.0, 8.0, -10.0, 10.0, 0.5)),
    (4, 5000, (-3.0, 4.5, -2.0, 2.0, -1.0, 1.0, 0.25)),
]

#: (seed, C, src grid, dst grid) of the pinned resampling cases
RESAMPLE_CASES = [
    (11, 3, (-51.2, 51.2, -51.2, 51.2, -10.0, 10.0, 0.8), (-54.0, 54.0, -54.0, 54.0, -10.0, 10.0, 0.3)),
    (12, 5, (-54.0, 54.0, -54.0, 54.0, -10.0, 10.0, 0.3), (-51.2, 51.2, -51.2, 51.2, -10.0, 10.0, 0.4)),
    (13, 2, (-8.0, 8.0, -8.0, 8.0, -5.0, 5.0, 0.5), (-10.0, 6.0, -7.5, 9.0, -5.0, 5.0, 0.25)),
    (14, 4, (-4.0, 4.0, -4.0, 4.0, -1.0, 1.0, 1.0), (-4.0, 4.0, -4.0, 4.0, -1.0, 1.0, 1.0)),
]


def random_map(seed: int, C: int, nx: int, ny: int) -> np.ndarray:
    return np.random.default_rng(seed).uniform(-1, 1, size=(C, nx, ny)).astype(np.float32)


def grid_shape(grid: tuple) -> tuple[int, int]:
    return (int(round((grid[1] - grid[0]) / grid[6])), int(round((grid[3] - grid[2]) / grid[6])))
