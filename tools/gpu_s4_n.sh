cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -3 gpurun_out/smoke.log
for c in C1 C2 C4; do
timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err
python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); r=d['roofline']; print('$c', round(d['value'],4), round(d['ms_per_step'],4), 'kern', round(r['kernel_ms_per_step'],3), 'frac', round(r['frac'],3), r.get('frac_sustained'), d['clocks']['sm_mhz'], d['u'], 'e2e', d['e2e']['value'], 'replayed', d['graph_replayed_steps'], 'strict', (d.get('fp64_strict') or {}).get('value'), 'cpu', (d.get('cpu_baseline') or {}).get('value'))"
done
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-strict --no-e2e > gpurun_out/s4n_C5.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/s4n_C5.json')); print('C5', round(d['ms_per_step']), d['clocks']['sm_mhz'], d['u'], d['graph_replayed_steps'])"
