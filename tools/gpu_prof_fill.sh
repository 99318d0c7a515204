CMD="python bench.py --steps 2 --warmup 1 --pairs 300000 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fill_kernel -s 1 -c 1 -o gpurun_out/fill_prof $CMD > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
