cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
for c in C3 C4; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-strict --no-e2e > gpurun_out/s4g_$c.json 2>gpurun_out/s4g_$c.err
python -c "
import json; d=json.load(open('gpurun_out/s4g_$c.json')); print('$c', round(d['value'],4), round(d['ms_per_step'],3), 'kern', round(d['roofline']['kernel_ms_per_step'],3), 'stream_ms', round(d['stream_ms_per_step'],3), d['clocks']['sm_mhz'], d['u'])"
done
CMD="python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-strict"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_C3.csv $CMD > gpurun_out/ncu_launch_C3.log 2>&1
python tools/launch_dram.py gpurun_out/r02_launches_C3.csv > gpurun_out/launches_C3.txt; head -16 gpurun_out/launches_C3.txt
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"stream_|sweep|finalize|pair_sym|zero_|oz_|ozaki_split|features|gram|sum_slices|times_small" --clock-control none --csv --log-file gpurun_out/r02_C5_stream_dram.csv python tools/c5_once.py > gpurun_out/ncu_c5_streams.log 2>&1
echo "== C5 rc=$?"; python tools/launch_dram.py gpurun_out/r02_C5_stream_dram.csv > gpurun_out/launches_C5_streams.txt; head -24 gpurun_out/launches_C5_streams.txt; tail -1 gpurun_out/launches_C5_streams.txt
