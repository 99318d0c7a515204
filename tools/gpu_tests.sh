# usage: bash tools/gpu_tests.sh [pytest -k expr]
K=${1:-}
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 240 -k "$K" > gpurun_out/pytest_gpu.log 2>&1
else
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 240 > gpurun_out/pytest_gpu.log 2>&1
fi
grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_gpu.log | tail -30
