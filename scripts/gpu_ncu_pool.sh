# ncu --set full of the interval kernels (S config).  Usage: bash scripts/gpu_ncu_pool.sh [which] [regex]
WHICH=${1:-fast}
RE=${2:-"pool_(slice|tile)_kernel"}
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$RE" -c 2 -o gpurun_out/prof_$WHICH -f python scripts/prof_pool.py $WHICH 1 > gpurun_out/ncu_$WHICH.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_$WHICH.log
