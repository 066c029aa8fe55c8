cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
USTATS_SCHED_DEBUG=1 timeout 1800 python tools/run_c5.py 65536 > gpurun_out/c5_full.log 2>&1; echo "c5 rc=$?"; grep -v "^\[alloc\]\|^\[free\]" gpurun_out/c5_full.log | tail -5; grep "^\[alloc\]\|^\[free\]\|sched" gpurun_out/c5_full.log | head -60
