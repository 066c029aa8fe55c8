cd $GRAFT_REPO_ROOT
for c in C2 C3 C4; do for cfg in "1 1" "1 0" "0 0"; do set -- $cfg
USTATS_OZ2_PERSIST=$1 USTATS_OZ2_LOCKSTEP=$2 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-strict --no-e2e > gpurun_out/ps_${c}_$1_$2.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/ps_${c}_$1_$2.json')); print('$c persist=$1 lockstep=$2', round(d['value'],2), round(d['ms_per_step'],2), 'gemm', round(d['roofline']['kernel_ms_per_step'],2), d['clocks']['sm_mhz'])"
done; done
