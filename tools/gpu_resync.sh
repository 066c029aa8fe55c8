cd $GRAFT_REPO_ROOT
for r in 1 0; do
USTATS_OZ2_RESYNC=$r timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-strict --no-e2e > gpurun_out/rs_$r.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/rs_$r.json')); print('resync=$r', round(d['ms_per_step']), 'gemm', round(d['roofline']['kernel_ms_per_step']), d['clocks']['sm_mhz'], d['u'])"
done
USTATS_OZ2_RESYNC=1 timeout 300 python tools/oz2_check.py 2>&1 | tail -3
