cd $GRAFT_REPO_ROOT
CMD="python bench.py --config ${CFG:-C2} --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_sw.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep -c 1 -o gpurun_out/sweep_full $CMD > gpurun_out/ncu_sweep.log 2>&1
echo "rc=$?"
