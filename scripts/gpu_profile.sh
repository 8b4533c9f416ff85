# Round profiling pass (one GPU): launch list of the bench command + ncu --set full of the S-config kernels.
# Usage: bash scripts/gpu_profile.sh [tag]
TAG=${1:-r01}
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu_$TAG.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -c 40 -o gpurun_out/prof_$TAG -f python scripts/prof_pool.py all 1 > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_$TAG.log
