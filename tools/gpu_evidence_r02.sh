# Round-2 final evidence: the default bench line, then the ncu launch list of the same
# command (cold-cache, serialised: shares, not absolute times).
python bench.py > gpurun_out/r02f_bench.log 2>&1; tail -1 gpurun_out/r02f_bench.log > gpurun_out/r02f_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_launches.csv python bench.py > gpurun_out/r02f_ncu_launch.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02f_smoke.log 2>&1
tail -1 gpurun_out/r02f_smoke.log
