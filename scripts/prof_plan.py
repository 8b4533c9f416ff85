"""The tile plan build from the association (bvp_build_tile_plan_ranks) at a
config, three times after a warm-up, for an ncu launch list:

    ncu --metrics gpu__time_duration.sum python scripts/prof_plan.py [S|H]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_13542_b200 as bp  # noqa: E402
from paper_2205_13542_b200.bevgrid import TilePlan  # noqa: E402

spec = bp.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "S"]
f = spec.frustum
rig, _, _, grid = bp.gen_workload(spec)
cache = bp.build_cache(rig, f, grid)
tp = TilePlan(spec.n_cameras, f.height, f.width, f.depth_bins, grid.n_cells, torch.device("cuda"))
for _ in range(4):
    tp.build(cache.d_cell_of_point, ranks=cache.d_ranks, counts=cache.d_counts)
torch.cuda.synchronize()
