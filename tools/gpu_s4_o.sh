cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "generated_rbf or graph_replay" > gpurun_out/gpu_tests_o.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/gpu_tests_o.log
timeout 900 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline --no-strict > gpurun_out/s4o_C1.json 2>gpurun_out/s4o_C1.err; tail -3 gpurun_out/s4o_C1.err
python -c "
import json; d=json.load(open('gpurun_out/s4o_C1.json')); print('C1', round(d['value'],4), round(d['ms_per_step'],4), 'kern', round(d['roofline']['kernel_ms_per_step'],4), d['clocks']['sm_mhz'], d['u'], 'e2e', d['e2e']['value'], d['graph_replayed_steps'], d['gpu_launches'])"
python tools/host_overhead.py 2>&1 | grep -v trace | tail -3
