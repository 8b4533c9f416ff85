# Round evidence on one GPU: tests, the B200-host reference probe, bench lines,
# launch list, ncu --set full of the headline kernels, sanitizers.
# Usage: bash scripts/gpu_round.sh <tag>
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=600 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 $OUT/pytest_gpu.log
PYTHONPATH=baseline/_ref OPENBLAS_NUM_THREADS=1 timeout 900 python tests/ref_host_probe.py $OUT/ref_host > $OUT/ref_host.log 2>&1; echo "probe rc=$?"
timeout 600 python bench.py --steps 30 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_reference.json 2>> $OUT/bench.err; echo "ref rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-variants > $OUT/bench_under_ncu.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:tile_pool_kernel|tile_finalize_kernel" -s 2 -c 2 -o $OUT/prof -f python scripts/prof_tile.py > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
bash scripts/sanitize_all.sh $OUT/san
(python scripts/time_fused_train.py 1; python scripts/time_fused_train.py 4; python scripts/time_train.py 4) > $OUT/train_timings.txt 2>&1; echo "train timings rc=$?"
for v in f32 fused; do ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -k regex:tile_ --csv python scripts/prof_tile_bwd.py $v 2>/dev/null | grep '^"' > $OUT/bwd_launch_$v.csv; done
ls -la $OUT
