# ncu captures of the S-config kernels (one GPU).  Usage: bash scripts/gpu_prof.sh
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pool_tile_kernel -c 6 -o gpurun_out/prof_pool -f python scripts/prof_pool.py all 1 > gpurun_out/ncu_pool.log 2>&1; echo "ncu rc=$?"
tail -5 gpurun_out/ncu_pool.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-variants --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1; echo "launches rc=$?"
