"""Regenerate tests/golden/ from the reference implementation itself.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_golden.py

It imports the reference ``bevpool`` package and records, for every BASELINE
configuration (T, S, H at seed 0) and for the seeded random instances the
reference's own tests use, SHA-256 digests of the reference's outputs:
cell_of_point / ranks / interval_starts / interval_cells (build_cache,
bevgrid.py:183-203), the depth softmax (normalize_depth, lift.py:17-31) and
pool_interval SUM / MEAN / MAX (pooling.py:206-221).  The T configuration's
index arrays are also stored in full (golden_T.npz).

The committed golden.json is what tests/ compare the oracle and the CUDA path
against; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))          # tests/
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))  # repo root

import bevpool as ref  # noqa: E402  (the reference, via PYTHONPATH)

from instances import GOLDEN_INSTANCES, random_instance  # noqa: E402
from oracle.oracle import CONFIGS  # noqa: E402  (config table only)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rig_from_rows(cams):
    return [ref.CameraCalibration(fx=r[0], fy=r[1], cx=r[2], cy=r[3],
                                  rotation=r[4:13].reshape(3, 3),
                                  translation=r[13:16], camera_id=i)
            for i, r in enumerate(cams)]


def record(rig, frustum, grid, features, logits):
    dist = ref.normalize_depth(logits)
    cache = ref.build_cache(rig, frustum, grid)
    entry = {
        "n_points": int(cache.n_points),
        "n_in": int(cache.n_in_range),
        "n_int": int(cache.n_intervals),
        "nx": int(grid.nx), "ny": int(grid.ny),
        "fingerprint": int(cache.fingerprint),
        "sha256": {
            "cell_of_point": sha(cache.cell_of_point.astype("<u4")),
            "ranks": sha(cache.ranks.astype("<u4")),
            "interval_starts": sha(cache.interval_starts.astype("<u4")),
            "interval_cells": sha(cache.interval_cells.astype("<u4")),
            "dist": sha(dist.astype("<f4")),
        },
    }
    for red in ref.Reducer:
        out = ref.pool_interval(features, dist, cache, grid, red)
        entry["sha256"][f"pool_{red.value}"] = sha(out.values.astype("<f4"))
        entry[f"pool_{red.value}_abs_sum"] = float(np.abs(out.values.astype(np.float64)).sum())
    return entry, cache


def main():
    golden = {"generated_by": "tests/golden/make_golden.py",
              "reference": "/root/reference/pkg/src/bevpool",
              "numpy": np.__version__, "configs": {}, "instances": {}}
    for name, cfg in CONFIGS.items():
        t0 = time.time()
        frustum = ref.FrustumSpec(cfg.height, cfg.width, cfg.depth_min,
                                  cfg.depth_step, cfg.depth_bins)
        grid = ref.BevGridSpec(*cfg.grid)
        spec = ref.WorkloadSpec(cfg.n_cameras, frustum, grid, cfg.channels, 0)
        rig, features, logits, _ = ref.gen_workload(spec)
        entry, cache = record(rig, frustum, grid, features, logits)
        entry["sha256"]["features"] = sha(features)
        entry["sha256"]["logits"] = sha(logits)
        golden["configs"][name] = entry
        if name == "T":
            np.savez_compressed(os.path.join(HERE, "golden_T.npz"),
                                cell_of_point=cache.cell_of_point,
                                ranks=cache.ranks,
                                interval_starts=cache.interval_starts,
                                interval_cells=cache.interval_cells)
        print(name, entry["n_in"], entry["n_int"], f"{time.time() - t0:.1f}s")

    # the restated instance generator must reproduce the reference suite's
    sys.path.insert(0, "/root/reference/pkg/tests")
    import conftest as ref_conftest  # noqa: E402
    for seed, mhw, md, mc in GOLDEN_INSTANCES:
        inst = random_instance(seed, mhw, md, mc)
        rig, frustum, grid, features, dist, cache = ref_conftest.random_instance(seed, mhw, md, mc)
        assert np.array_equal(features, inst.features), seed
        assert (grid.nx, grid.ny) == (inst.nx, inst.ny), seed
        assert tuple(grid.__dict__[k] for k in ("x_min", "x_max", "y_min", "y_max", "z_min", "z_max", "r")) == inst.grid
        for cam, row in zip(rig, inst.cams):
            assert np.array_equal(cam.rotation.reshape(-1), row[4:13])
            assert np.array_equal(cam.translation, row[13:16])
            assert (cam.fx, cam.fy, cam.cx, cam.cy) == tuple(row[:4])
        entry, _ = record(rig_from_rows(inst.cams), frustum, grid, features, inst.logits)
        golden["instances"][str(seed)] = entry
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(golden, fh, indent=1, sort_keys=True)
    print("wrote", len(golden["instances"]), "instances")


if __name__ == "__main__":
    main()
