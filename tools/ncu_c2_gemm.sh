# full ncu capture of the C2 fused symmetric GEMM (main phase) of one step
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_gemm.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_tma -s 0 -c 1 -o gpurun_out/c2_gemm_full $CMD > gpurun_out/ncu_c2_gemm.log 2>&1
echo "full rc=$?"
