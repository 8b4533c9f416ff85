# Round evidence on one GPU: tests, bench line, launch list, ncu --set full of the
# dominant kernels, gather ceiling microbenchmark.  Usage: bash scripts/gpu_round.sh <tag>
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=300 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_reference.json 2>> $OUT/bench.err; echo "ref rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_under_ncu.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:pool_ivl_kernel|pixel_softmax" -c 3 -o $OUT/prof -f python scripts/prof_pool.py all 1 > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gmlp scripts/gather_mlp_bench.cu && /tmp/gmlp > $OUT/gather_mlp_bench.txt 2>&1
ls -la $OUT
timeout 300 python scripts/time_train.py 4 > $OUT/train.txt 2>&1
timeout 300 python scripts/time_assoc.py S H > $OUT/assoc.txt 2>&1
timeout 900 python scripts/stage_compare.py > $OUT/stages.txt 2>&1
timeout 300 python scripts/time_zero.py > $OUT/zero_fill.txt 2>&1
