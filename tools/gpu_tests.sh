# usage: bash tools/gpu_tests.sh [pytest -k expr]
K=${1:-}
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "$K" > gpurun_out/pytest_gpu.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
fi
grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_gpu.log | tail -30
