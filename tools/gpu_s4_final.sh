# final-tree evidence: GPU tests, smoke, the driver's default bench line (C5), the reference arm, C1-C4 lines
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -3 gpurun_out/smoke.log
/usr/bin/time -v timeout 2400 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
grep -E "Elapsed|Maximum resident" gpurun_out/bench_default.err
python -c "
import json; d=json.load(open('gpurun_out/bench_default.json')); r=d['roofline']; print('C5', d['value'], d['ms_per_step'], r['frac'], r.get('frac_sustained'), r['kernel_ms_per_step'], d['clocks'], (d.get('e2e') or {}).get('value'), (d.get('fp64_strict') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'))"
timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"; head -c 700 gpurun_out/bench_reference.json; echo
for c in C1 C2 C3 C4; do
timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err
python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); r=d['roofline']; print('$c', round(d['value'],4), round(d['ms_per_step'],3), 'kern', round(r['kernel_ms_per_step'],3), 'frac', round(r['frac'],3), r.get('frac_sustained'), 'stream_ms', round(d['stream_ms_per_step'],3), d['clocks']['sm_mhz'], d['u'], 'e2e', d['e2e']['value'], 'strict', (d.get('fp64_strict') or {}).get('value'), 'cpu', (d.get('cpu_baseline') or {}).get('value'))"
done
