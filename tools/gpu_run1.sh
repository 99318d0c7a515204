nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
./paper_2002_04561_b200/lib/dpx_bench > gpurun_out/dpx.json 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/dpx.json; tail -3 gpurun_out/bench.log; cat gpurun_out/smoke.log | tail -3
