# round-2 evidence: GPU tests, smoke, the driver's default bench line (C5),
# the reference arm, the C2 line, ncu captures of the CTA-pair GEMM
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -3 gpurun_out/smoke.log
/usr/bin/time -v timeout 2400 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
grep -E "Elapsed|Maximum resident" gpurun_out/bench_default.err
python -c "
import json; d=json.load(open('gpurun_out/bench_default.json')); print('C5', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms_per_step'], d['clocks'], (d.get('e2e') or {}).get('value'), (d.get('fp64_strict') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'))"
timeout 1200 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"; cat gpurun_out/bench_reference.json | head -c 600; echo
timeout 600 python bench.py --config C2 --steps 20 --warmup 5 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; echo "c2 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ozaki_gemm_2sm -c 1 -o gpurun_out/r02_C2_oz2sm python bench.py --config C2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-strict > gpurun_out/ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second -k regex:ozaki_gemm_2sm -s 4 -c 3 --clock-control none --csv --log-file gpurun_out/r02_C5_oz2sm_metrics.csv python tools/c5_once.py > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
