# round 2 first check: GPU tests, smoke, C5 headline through bench.py
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -15 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -3 gpurun_out/smoke.log
USTATS_SCHED_DEBUG=1 timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-strict > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_C5.json; grep -v "^\[alloc\]\|^\[free\]" gpurun_out/bench_C5.err | tail -20
