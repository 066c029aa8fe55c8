cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q -k "C4_n512" > gpurun_out/gpu_tests_l.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/gpu_tests_l.log
