cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
for c in C1 C2 C4; do
timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-strict > gpurun_out/s4j_$c.json 2>gpurun_out/s4j_$c.err
python -c "
import json; d=json.load(open('gpurun_out/s4j_$c.json')); print('$c', round(d['value'],4), round(d['ms_per_step'],4), 'kern', round(d['roofline']['kernel_ms_per_step'],3), 'stream_ms', round(d['stream_ms_per_step'],3), d['clocks']['sm_mhz'], d['u'], 'e2e', d['e2e']['value'])"
done
python tools/host_overhead.py 2>&1 | grep -v trace | tail -3
