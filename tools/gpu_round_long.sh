# ncu summaries of the secondary kernels: long kernel (C4 shape, 1.2 Mbp, local affine) and the
# traceback fill + walk (C3 shape, 300k pairs).  Each command runs plain first.
python tools/long_one.py 1200000 > gpurun_out/l1.log 2>&1 && \
ncu --section WarpStateStats --section SourceCounters --section SchedulerStats --section LaunchStats \
    --section Occupancy --section MemoryWorkloadAnalysis --section SpeedOfLight \
    --metrics sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:long_kernel -c 1 -o gpurun_out/long_r01 python tools/long_one.py 1200000 > gpurun_out/ncu_long.log 2>&1
tail -1 gpurun_out/ncu_long.log
