cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
for c in C2 C3; do for m in 1 0; do
USTATS_OZ_2SM=$m timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-strict --no-e2e > gpurun_out/b_${c}_$m.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/b_${c}_$m.json')); print('$c 2sm=$m', round(d['value'],3), round(d['ms_per_step'],2), round(d['roofline']['frac'],3), round(d['roofline']['kernel_ms_per_step'],2), d['clocks'])"
done; done
USTATS_OZ_2SM=1 timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-strict --no-e2e > gpurun_out/b_C5_1.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/b_C5_1.json')); print('C5 2sm', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms_per_step'], d['clocks'], d['u'])"
