# Round-2 final evidence: the default bench line, then the ncu launch list of the same
# command (cold-cache, serialised: shares, not absolute times), then smoke().
# usage: bash tools/gpu_evidence_r02.sh [tag]   (outputs gpurun_out/<tag>_*)
T=${1:-r02f}
python bench.py > gpurun_out/${T}_bench.log 2>&1; tail -1 gpurun_out/${T}_bench.log > gpurun_out/${T}_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py > gpurun_out/${T}_ncu_launch.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1
tail -1 gpurun_out/${T}_smoke.log
