# iteration loop: GPU parity tests + quick bench lines
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x -v 2>&1 | grep -v "^  File" | grep -v PASSED | tail -25
for c in C2 C1 C3 C4; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "
import json,sys; d=json.load(open('gpurun_out/bench_$c.json'))
print('$c', 'value %.4g evals/s'%d['value'], 'ms %.3f'%d['ms_per_step'], 'e2e %.4g'%d.get('e2e',{}).get('value',0), 'roof %s %.3g %.3f'%(d['roofline']['unit'], d['roofline']['achieved'] or 0, d['roofline']['frac'] or 0), 'gemm_ms %.2f'%d['roofline']['kernel_ms_per_step'], 'stream_ms %.2f'%d['stream_ms_per_step'], d['stats_per_step'], 'u', d['u'])
" || tail -5 gpurun_out/bench_$c.err
done
