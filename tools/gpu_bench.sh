# bench sweep on one B200: default line (C2) + the other single-GPU configs
set -x
cd $GRAFT_REPO_ROOT
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
for c in C1 C3 C4; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
cat gpurun_out/bench_*.json
tail -5 gpurun_out/bench_*.err
