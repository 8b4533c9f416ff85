python scripts/time_tile.py S 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tile_pool python scripts/fused_prof.py 2>&1 | grep -E "duration" | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tile_pool python scripts/prof_tile.py 2>&1 | grep -E "duration" | tail -1
