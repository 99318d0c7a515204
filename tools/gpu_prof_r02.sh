# Round-2 evidence: the bench line, its ncu launch list, and full captures of the top kernels
# (each command first runs plain; a number printed under ncu is never a bench value).
set -x
python bench.py > gpurun_out/r02_bench.log 2>&1; tail -1 gpurun_out/r02_bench.log > gpurun_out/r02_bench.json
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv $CMD > gpurun_out/r02_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fill_kernel -s 3 -c 1 -o gpurun_out/r02_fill $CMD --long-bp 0 --long-tb-bp 0 > gpurun_out/r02_ncu_fill.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:long16 -c 1 -o gpurun_out/r02_long16 python tools/long_one.py 1200000 296 0 1 > gpurun_out/r02_ncu_long16.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"fill_kernel|walk_kernel" -s 2 -c 2 -o gpurun_out/r02_tbfill python tools/tb8_probe.py 100000 1 1 > gpurun_out/r02_ncu_tb.log 2>&1
ls -la gpurun_out/ | tail -12
