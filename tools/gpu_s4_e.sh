cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline --no-strict > gpurun_out/s4e_C3.json 2>gpurun_out/s4e_C3.err
python -c "
import json; d=json.load(open('gpurun_out/s4e_C3.json')); print('C3', round(d['value'],4), round(d['ms_per_step'],3), 'kern', round(d['roofline']['kernel_ms_per_step'],3), d['clocks']['sm_mhz'], d['u'])"
SECONDS=0
timeout 2400 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$? wall ${SECONDS}s"
python -c "
import json; d=json.load(open('gpurun_out/bench_default.json')); r=d['roofline']; print('C5', d['value'], d['ms_per_step'], r['frac'], r.get('frac_sustained'), r['kernel_ms_per_step'], d['clocks'], (d.get('e2e') or {}).get('value'), (d.get('fp64_strict') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'))"
