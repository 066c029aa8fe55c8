cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
for c in C3 C4; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-strict --no-e2e > gpurun_out/xp_$c.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/xp_$c.json')); r=d['roofline']; print('$c', round(d['value'],3), round(d['ms_per_step'],3), r['bound'], round(r['frac'],3), round(d['stream_ms_per_step'],3), d['clocks']['sm_mhz'], d['stats_per_step']['executed_stream_entries'])"
done
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-strict --no-e2e > gpurun_out/xp_C5.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/xp_C5.json')); print('C5', round(d['ms_per_step']), round(d['stream_ms_per_step']), d['clocks']['sm_mhz'], d['u'])"
