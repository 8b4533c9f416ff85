"""Run the unmodified reference on THIS host and digest its outputs.

    PYTHONPATH=baseline/_ref OPENBLAS_NUM_THREADS=1 python tests/ref_host_probe.py OUT_DIR

Used by tests/test_ref_host.py on the GPU box (where /root/reference does
not exist, but baseline/_ref -- the reference installed unmodified -- does).
For configs T, S and H (seed 0) it records the same SHA-256 digests as
tests/golden/make_golden.py (build_cache arrays, normalize_depth, the three
pool_interval reducers), plus, for T and S, the reference's own dist and SUM
map as .npy files so the CUDA path can be fed and checked on the very same
host.  The reference's arithmetic depends on the host: the frustum goes
through OpenBLAS dgemm (geometry.py:185, DYNAMIC_ARCH picks a kernel per
CPU) and the softmax through numpy's SIMD exp (lift.py:28-31); this probe is
how a B200 host's results are pinned against the build container's goldens.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

import bevpool as ref  # the reference (baseline/_ref on PYTHONPATH)

CONFIGS = {  # SURVEY.md §8 config table (same as oracle.CONFIGS)
    "T": (1, 16, 44, 1.0, 1.0, 59, 32, (-51.2, 51.2, -51.2, 51.2, -10.0, 10.0, 0.8)),
    "S": (6, 32, 88, 1.0, 0.5, 118, 80, (-54.0, 54.0, -54.0, 54.0, -10.0, 10.0, 0.3)),
    "H": (6, 64, 176, 1.0, 0.5, 118, 80, (-54.0, 54.0, -54.0, 54.0, -10.0, 10.0, 0.15)),
}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main(out_dir: str) -> None:
    os.makedirs(out_dir, exist_ok=True)
    res = {"numpy": np.__version__, "cpu_count": os.cpu_count(), "configs": {}}
    try:
        res["cpu"] = next(ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo")
                          if ln.startswith("model name"))
    except (OSError, StopIteration):
        res["cpu"] = "?"
    for name, (n, h, w, dmin, dstep, d, c, grid) in CONFIGS.items():
        frustum = ref.FrustumSpec(h, w, dmin, dstep, d)
        g = ref.BevGridSpec(*grid)
        rig, features, logits, _ = ref.gen_workload(ref.WorkloadSpec(n, frustum, g, c, 0))
        dist = ref.normalize_depth(logits)
        cache = ref.build_cache(rig, frustum, g)
        e = {"n_in": int(cache.n_in_range), "n_int": int(cache.n_intervals), "sha256": {
            "cell_of_point": sha(cache.cell_of_point.astype("<u4")),
            "ranks": sha(cache.ranks.astype("<u4")),
            "interval_starts": sha(cache.interval_starts.astype("<u4")),
            "interval_cells": sha(cache.interval_cells.astype("<u4")),
            "dist": sha(dist.astype("<f4")),
        }}
        for red in ref.Reducer:
            out = ref.pool_interval(features, dist, cache, g, red)
            e["sha256"][f"pool_{red.value}"] = sha(out.values.astype("<f4"))
            if name != "H" and red is ref.Reducer.SUM:
                np.save(os.path.join(out_dir, f"{name}_pool_sum.npy"), out.values)
        if name != "H":
            np.save(os.path.join(out_dir, f"{name}_dist.npy"), dist)
        res["configs"][name] = e
    with open(os.path.join(out_dir, "ref_host.json"), "w") as fh:
        json.dump(res, fh, indent=1, sort_keys=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main(sys.argv[1])
