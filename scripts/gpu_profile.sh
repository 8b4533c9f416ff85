# Round profiling pass (one GPU): launch list of the bench command + ncu --set full of the S-config kernels.
# Usage: bash scripts/gpu_profile.sh [tag] [kernel-regex] [count]
TAG=${1:-r01}
RE=${2:-"pool_unit_kernel|pool_long_kernel|pixel_lse|lift"}
CNT=${3:-8}
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu_$TAG.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$RE" -c $CNT -o gpurun_out/prof_$TAG -f python scripts/prof_pool.py all 1 > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_$TAG.log
ls -la gpurun_out/
