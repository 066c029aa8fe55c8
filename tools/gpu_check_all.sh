cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
for c in C5 C4; do
timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-strict --no-e2e > gpurun_out/chk_$c.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/chk_$c.json')); print('$c', round(d['value'],4), round(d['ms_per_step'],2), 'gemm', round(d['roofline']['kernel_ms_per_step'],2), d['clocks']['sm_mhz'], d['u'], d['stats_per_step']['executed_stream_entries'])"
done
