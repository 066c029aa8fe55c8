# launch lists (serialized, cold) of one evaluation of C1/C3/C4 + DRAM counters of every C5 stream kernel
cd $GRAFT_REPO_ROOT
for CFG in C1 C3 C4; do
  CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-strict"
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_$CFG.csv $CMD > gpurun_out/ncu_launch_$CFG.log 2>&1
  echo "== $CFG rc=$?"
done
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"stream_|sweep|finalize|pair_sym|zero_|oz_|ozaki_split|features|gram|sum_slices" --clock-control none --csv --log-file gpurun_out/r02_C5_stream_dram.csv python tools/c5_once.py > gpurun_out/ncu_c5_streams.log 2>&1
echo "== C5 rc=$?"; tail -2 gpurun_out/ncu_c5_streams.log
USTATS_TRACE=1 python tools/host_overhead.py 2>&1 | tail -20
