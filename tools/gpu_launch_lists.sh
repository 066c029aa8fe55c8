# launch lists (serialized, cold) of one evaluation per config + C5 GEMM counters
cd $GRAFT_REPO_ROOT
for CFG in C1 C3 C4; do
  CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-strict"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_launch_$CFG.log 2>&1
  echo "== $CFG rc=$?"; python tools/launch_summary.py gpurun_out/launches_$CFG.csv 2>&1 | head -14
done
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-strict"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file gpurun_out/launches_C5.csv $CMD > gpurun_out/ncu_launch_C5.log 2>&1
echo "== C5 rc=$?"
