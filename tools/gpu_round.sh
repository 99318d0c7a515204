# round measurement, call 1: microbench, bench (default command, plain), secondary configs,
# then the launch list of the same bench command under ncu (one ncu tool per call)
set -x
./paper_2002_04561_b200/lib/dpx_bench > gpurun_out/dpx.json 2> gpurun_out/dpx.err
bash tools/build_tools.sh && ./tools/bin/pipebench > gpurun_out/pipebench.txt 2>&1
CMD="python bench.py"
$CMD > gpurun_out/bench_full.log 2>&1
tail -1 gpurun_out/bench_full.log
python tools/bench_configs.py > gpurun_out/configs.log 2>&1
tail -8 gpurun_out/configs.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
tail -1 gpurun_out/ncu_launch.log | cut -c1-200
