cd $GRAFT_REPO_ROOT
USTATS_OZ2_SYMG=2 USTATS_OZ2_GROUP=2 timeout 300 python tools/oz2_check.py 2>&1 | tail -10
USTATS_OZ2_SYMG=3 timeout 300 python tools/oz2_check.py 2>&1 | head -7
for cfg in "2 0" "2 2" "2 1" "2 4"; do set -- $cfg
USTATS_OZ2_GROUP=$1 USTATS_OZ2_SYMG=$2 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-strict --no-e2e > gpurun_out/l2b_$1_$2.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/l2b_$1_$2.json')); print('group=$1 symg=$2', round(d['ms_per_step']), 'gemm', round(d['roofline']['kernel_ms_per_step']), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['u'])"
done
