cd $GRAFT_REPO_ROOT
mode=${1:-wavefront}
python scripts/wcycle_launches.py 12 w $mode > gpurun_out/wfl_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/wfl_launches_$mode.csv python scripts/wcycle_launches.py 12 w $mode > gpurun_out/wfl_ncu.log 2>&1
