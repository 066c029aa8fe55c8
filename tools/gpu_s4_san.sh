cd $GRAFT_REPO_ROOT
timeout 1700 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -5 gpurun_out/sanitize_memcheck.log
