cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q -k "ozaki or emulat or lazy or C4 or khatri or golden or dgemm" > gpurun_out/gpu_tests_d.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gpu_tests_d.log
for c in C2 C3 C4; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-strict > gpurun_out/s4d_$c.json 2>gpurun_out/s4d_$c.err
python -c "
import json; d=json.load(open('gpurun_out/s4d_$c.json')); print('$c', round(d['value'],4), round(d['ms_per_step'],3), 'kern', round(d['roofline']['kernel_ms_per_step'],3), 'frac', round(d['roofline']['frac'],3), round(d['roofline']['frac_sustained'],3), 'stream_ms', round(d['stream_ms_per_step'],3), d['clocks']['sm_mhz'], d['u'])"
done
CMD="python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-strict"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_C4.csv $CMD > gpurun_out/ncu_launch_C4.log 2>&1
python tools/launch_dram.py gpurun_out/r02_launches_C4.csv > gpurun_out/launches_C4.txt; head -12 gpurun_out/launches_C4.txt
CMD="python bench.py --config C2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-strict"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_C2.csv $CMD > gpurun_out/ncu_launch_C2.log 2>&1
python tools/launch_dram.py gpurun_out/r02_launches_C2.csv > gpurun_out/launches_C2.txt; head -12 gpurun_out/launches_C2.txt
