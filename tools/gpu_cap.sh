cd $GRAFT_REPO_ROOT
for cap in 4 8 16; do
USTATS_OZ_DIGIT_CAP_GB=$cap timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline --no-strict --no-e2e > gpurun_out/cap_C4_$cap.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/cap_C4_$cap.json')); print('C4 cap=$cap', round(d['value'],3), round(d['ms_per_step'],1), 'gemm', round(d['roofline']['kernel_ms_per_step'],1), d['roofline']['frac'], d['clocks']['sm_mhz'], d['u'])"
done
for cap in 8 4; do
USTATS_OZ_DIGIT_CAP_GB=$cap timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-strict --no-e2e > gpurun_out/cap_C5_$cap.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/cap_C5_$cap.json')); print('C5 cap=$cap', round(d['ms_per_step']), 'gemm', round(d['roofline']['kernel_ms_per_step']), d['clocks']['sm_mhz'], d['u'])"
done
