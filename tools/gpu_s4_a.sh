# session check: GPU tests, smoke, short bench lines of all five configs
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -3 gpurun_out/smoke.log
for c in C1 C2 C3 C4 C5; do
st=10; [ $c = C5 ] && st=2
timeout 900 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --no-strict > gpurun_out/s4_$c.json 2>gpurun_out/s4_$c.err
python -c "
import json; d=json.load(open('gpurun_out/s4_$c.json')); print('$c', round(d['value'],4), round(d['ms_per_step'],3), 'kern', round(d['roofline']['kernel_ms_per_step'],3), 'frac', round(d['roofline']['frac'],3), 'stream_ms', round(d['stream_ms_per_step'],3), d['clocks']['sm_mhz'], d['u'], d['stats_per_step']['executed_stream_entries'], 'e2e', d['e2e']['value'])"
done
