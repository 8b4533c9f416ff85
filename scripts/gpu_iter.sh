# quick iteration: gpu tests + per-kernel timings.  Usage: bash scripts/gpu_iter.sh [pytest -k expr]
K=${1:-}
if [ -n "$K" ]; then KARG="-k $K"; else KARG=""; fi
timeout 900 python -m pytest tests -m gpu -q --maxfail=10 -p no:cacheprovider --timeout=300 $KARG > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|Error" gpurun_out/pytest_gpu.log | tail -15
timeout 300 python scripts/time_kernels.py 20 2>&1 | tail -12
