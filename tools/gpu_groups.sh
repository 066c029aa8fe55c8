cd $GRAFT_REPO_ROOT
for g in 4 12 16; do
USTATS_OZ2_GROUP=$g USTATS_OZ2_SYMG=$g timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-strict --no-e2e > gpurun_out/g_$g.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/g_$g.json')); print('G=$g', round(d['ms_per_step']), 'gemm', round(d['roofline']['kernel_ms_per_step']), d['clocks']['sm_mhz'], d['u'])"
done
