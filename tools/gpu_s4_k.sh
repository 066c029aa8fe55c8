cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q -k "ragged_small" > gpurun_out/gpu_tests_k.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/gpu_tests_k.log
