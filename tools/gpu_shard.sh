cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q -k "shard" > gpurun_out/shard_tests.log 2>&1; echo "shard rc=$?" >> gpurun_out/shard_tests.log
tail -30 gpurun_out/shard_tests.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
