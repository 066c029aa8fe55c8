cd $GRAFT_REPO_ROOT
for cfg in "8 0" "2 0" "2 1" "8 1" "3 1"; do set -- $cfg
USTATS_OZ2_GROUP=$1 USTATS_OZ2_HINT=$2 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-strict --no-e2e > gpurun_out/l2_$1_$2.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/l2_$1_$2.json')); print('group=$1 hint=$2', round(d['ms_per_step']), 'gemm', round(d['roofline']['kernel_ms_per_step']), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['u'])"
done
