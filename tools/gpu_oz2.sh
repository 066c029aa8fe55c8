cd $GRAFT_REPO_ROOT
export USTATS_OZ_2SM=1
timeout 180 python tools/oz2_check.py > gpurun_out/oz2_on.log 2>&1; echo "on rc=$?" >> gpurun_out/oz2_on.log
cat gpurun_out/oz2_on.log
USTATS_OZ_2SM=0 timeout 180 python tools/oz2_check.py > gpurun_out/oz2_off.log 2>&1; echo "off rc=$?" >> gpurun_out/oz2_off.log
cat gpurun_out/oz2_off.log
if grep -q "on rc=0" gpurun_out/oz2_on.log; then
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -5 gpurun_out/gpu_tests.log
timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-strict > gpurun_out/bench_C2.json 2>gpurun_out/bench_C2.err; echo "c2 rc=$?"
USTATS_OZ_2SM=0 timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline --no-strict > gpurun_out/bench_C2_1sm.json 2>gpurun_out/bench_C2_1sm.err
for f in bench_C2 bench_C2_1sm; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'])"; done
fi
