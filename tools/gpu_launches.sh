# launch list of one C2 step (cold, serialized) for share-of-step accounting
cd $GRAFT_REPO_ROOT
CFG=${CFG:-C2}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$CFG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_launch_$CFG.log 2>&1
echo "launches rc=$?"
