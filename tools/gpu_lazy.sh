cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_full.py -q -x -m gpu -k "lazy or C4" 2>&1 | tail -3
timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline --no-strict --no-e2e > gpurun_out/lazy_C4.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/lazy_C4.json')); print('C4', round(d['value'],3), round(d['ms_per_step'],1), 'gemm', round(d['roofline']['kernel_ms_per_step'],1), d['roofline']['frac'], d['clocks']['sm_mhz'], d['stats_per_step']['executed_stream_entries'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C4_lazy.csv python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-strict > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_C4_lazy.csv | head -12
