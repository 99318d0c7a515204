# launch list + one full capture of the fill kernel (run the same command plain first)
CMD="python bench.py --steps 2 --warmup 1 --pairs 200000 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 ; \
ncu --set full --clock-control none --import-source on -k regex:fill_kernel -s 1 -c 1 -o gpurun_out/fill_prof $CMD > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/prof_plain.log | cut -c1-300; tail -3 gpurun_out/ncu_full.log
