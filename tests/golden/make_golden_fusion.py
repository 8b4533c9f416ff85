"""Regenerate tests/golden/golden_fusion.json from the reference itself.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_golden_fusion.py

SHA-256 digests of the reference's lidar_to_bev (SUM / MEAN / MAX,
fusion.py:19-53) and grid_resample (fusion.py:70-108) on the seeded inputs of
tests/instances.py (LIDAR_CASES, RESAMPLE_CASES).  Nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import bevpool as ref  # noqa: E402  (the reference, via PYTHONPATH)

from instances import LIDAR_CASES, RESAMPLE_CASES, grid_shape, random_cloud, random_map  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out = {"generated_by": "tests/golden/make_golden_fusion.py", "lidar": {}, "resample": {}}
    for seed, n, g in LIDAR_CASES:
        grid = ref.BevGridSpec(*g)
        pts = random_cloud(seed, n, g)
        e = {"points": sha(pts)}
        for red in ref.Reducer:
            m = ref.lidar_to_bev(pts, grid, red)
            e[red.value] = sha(m.values.astype("<f4"))
        out["lidar"][str(seed)] = e
    for seed, C, sg, dg in RESAMPLE_CASES:
        snx, sny = grid_shape(sg)
        src = ref.BevFeatureMap(random_map(seed, C, snx, sny), ref.BevGridSpec(*sg))
        m = ref.grid_resample(src, ref.BevGridSpec(*dg))
        out["resample"][str(seed)] = {"dst": sha(m.values.astype("<f4")),
                                      "shape": list(m.values.shape)}
    with open(os.path.join(HERE, "golden_fusion.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print("wrote", len(out["lidar"]), "lidar and", len(out["resample"]), "resample cases")


if __name__ == "__main__":
    main()
