# round measurement: microbench, bench (plain), launch list, full ncu capture of the fill kernel
set -x
./paper_2002_04561_b200/lib/dpx_bench > gpurun_out/dpx.json 2> gpurun_out/dpx.err
cp gpurun_out/dpx.json profiles/dpx_rates.json
CMD="python bench.py --steps 5 --warmup 3"
$CMD > gpurun_out/bench_full.log 2>&1
tail -1 gpurun_out/bench_full.log
CMD2="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$CMD2 > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD2 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fill_kernel -s 1 -c 1 -o gpurun_out/fill_full $CMD2 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
