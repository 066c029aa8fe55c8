cd $GRAFT_REPO_ROOT
timeout 300 python tools/oz2_check.py 2>&1 | tail -10
USTATS_OZ2_LOCKSTEP=0 timeout 300 python tools/oz2_check.py 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_dgemm.py tests/test_gpu_full.py -q -x -m gpu 2>&1 | tail -2
for cfg in "1 1" "1 0" "0 0"; do set -- $cfg
USTATS_OZ2_PERSIST=$1 USTATS_OZ2_LOCKSTEP=$2 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-strict --no-e2e > gpurun_out/ps_$1_$2.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/ps_$1_$2.json')); print('persist=$1 lockstep=$2', round(d['ms_per_step']), 'gemm', round(d['roofline']['kernel_ms_per_step']), d['clocks']['sm_mhz'], d['u'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second -k regex:ozaki_gemm_2sm -s 4 -c 2 --clock-control none --csv --log-file gpurun_out/ps_C5_metrics.csv python tools/c5_once.py > /dev/null 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/ps_C5_metrics.csv')) if len(r)>10]
h=rows[0]
for r in rows[1:]: print(r[h.index('ID')], r[h.index('Grid Size')], r[h.index('Metric Name')], r[h.index('Metric Value')])
PY
