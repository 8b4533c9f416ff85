"""Golden digests of the reference's generate_frustum / quantize_points.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_golden_frustum.py

Writes tests/golden/golden_frustum.json: for configs T and S (seed-0 rig)
the SHA-256 of the reference's frustum coordinates (geometry.py:162-191,
float64 (P, 3)) and of quantize_points over them (bevgrid.py:85-98), plus
the reference's own quantize KATs evaluated by the reference.
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import bevpool as ref  # noqa: E402
from oracle.oracle import CONFIGS  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out = {"generated_by": "tests/golden/make_golden_frustum.py", "configs": {}}
    for name in ("T", "S"):
        cfg = CONFIGS[name]
        frustum = ref.FrustumSpec(cfg.height, cfg.width, cfg.depth_min, cfg.depth_step,
                                  cfg.depth_bins)
        grid = ref.BevGridSpec(*cfg.grid)
        rig = ref.synthetic_rig(cfg.n_cameras, frustum)
        pts = ref.generate_frustum(rig, frustum)
        cells = ref.quantize_points(grid, pts.coords)
        out["configs"][name] = {"coords": sha(pts.coords.astype("<f8")),
                                "cells": sha(cells.astype("<u4")), "n_points": len(pts)}
    g = ref.DEFAULT_GRID
    kat = [[0.0, 0.0, 0.0], [51.2, 0.0, 0.0], [-51.2, -51.2, -10.0], [0.0, 0.0, 10.0],
           [0.0, 0.0, -10.0], [51.1999, 51.1999, 9.999], [-51.2, 0.4, 0.0], [0.4, -51.2, 0.0]]
    out["kat"] = {"points": kat, "cells": [int(c) for c in ref.quantize_points(g, np.array(kat))]}
    with open(os.path.join(HERE, "golden_frustum.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print(json.dumps(out["kat"]))


if __name__ == "__main__":
    main()
