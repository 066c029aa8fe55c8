cd $GRAFT_REPO_ROOT
START=$(date +%s)
timeout 2400 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$? wall=$(( $(date +%s) - START ))s"
python -c "
import json; d=json.load(open('gpurun_out/bench_default.json')); print('C5', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms_per_step'], d['clocks'], (d.get('e2e') or {}).get('value'), (d.get('fp64_strict') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'))"
tail -3 gpurun_out/bench_default.err
