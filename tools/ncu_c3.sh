cd $GRAFT_REPO_ROOT
CMD="python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_tma -s 1 -c 1 -o gpurun_out/c3_gemm $CMD > gpurun_out/ncu_c3.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_c3.log
