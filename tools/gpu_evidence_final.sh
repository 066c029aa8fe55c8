# final-tree evidence: GPU tests, smoke, the driver's default bench line (C5), the reference arm,
# C1-C4 lines, launch lists with DRAM bytes, ncu counters of the C5 GEMM chunk launches
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -3 gpurun_out/smoke.log
SECONDS=0
timeout 2400 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$? wall ${SECONDS}s"
python -c "
import json; d=json.load(open('gpurun_out/bench_default.json')); r=d['roofline']; print('C5', d['value'], d['ms_per_step'], r['frac'], r.get('frac_sustained'), r['kernel_ms_per_step'], d['clocks'], (d.get('e2e') or {}).get('value'), (d.get('fp64_strict') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'))"
SECONDS=0
timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$? wall ${SECONDS}s"; head -c 300 gpurun_out/bench_reference.json; echo
for c in C1 C2 C3 C4; do
timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err
python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); r=d['roofline']; print('$c', round(d['value'],4), round(d['ms_per_step'],4), 'kern', round(r['kernel_ms_per_step'],3), 'frac', round(r['frac'],3), r.get('frac_sustained'), 'stream_ms', round(d['stream_ms_per_step'],3), d['clocks']['sm_mhz'], d['u'], 'e2e', d['e2e']['value'], 'strict', (d.get('fp64_strict') or {}).get('value'), 'cpu', (d.get('cpu_baseline') or {}).get('value'))"
done
for CFG in C1 C2 C3 C4; do
  CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-strict"
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_$CFG.csv $CMD > gpurun_out/ncu_launch_$CFG.log 2>&1
  echo "== $CFG rc=$?"; python tools/launch_dram.py gpurun_out/r02_launches_$CFG.csv > gpurun_out/launches_$CFG.txt; head -8 gpurun_out/launches_$CFG.txt
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__m_xbar2l1tex_read_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
timeout 1500 ncu --metrics $M --clock-control none -k regex:ozaki_gemm_2sm -s 4 -c 3 --csv --log-file gpurun_out/r02_C5_oz2sm_final_metrics.csv python tools/c5_once.py > gpurun_out/c5_ncu.log 2>&1; echo "ncu c5 rc=$?"
tail -2 gpurun_out/c5_ncu.log
