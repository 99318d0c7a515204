# round measurement, call 2: one full ncu capture of the dominant kernel (fill) in the bench
# command (run plain first: ncu only after the same command exited 0 without it)
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fill_kernel -s 3 -c 1 -o gpurun_out/fill_full $CMD > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
