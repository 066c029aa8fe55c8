# end-of-session evidence: GPU tests, smoke, default bench line, reference arm, C2 launch list
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench_C2_default.json 2> gpurun_out/bench_C2_default.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_C2_reference.json 2> gpurun_out/bench_C2_reference.err
for c in C1 C3 C4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/C2_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1
tail -2 gpurun_out/gpu_tests.log; tail -1 gpurun_out/smoke.log
for c in C2_default C2_reference C1 C3 C4; do python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', d.get('value'), d.get('ms_per_step'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), d.get('clocks'))" || tail -3 gpurun_out/bench_$c.err; done
