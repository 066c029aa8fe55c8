cd $GRAFT_REPO_ROOT
python tools/gemm_probe.py 4096 2 > gpurun_out/gemm_probe.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_f64 -s 0 -c 1 -o gpurun_out/gemm_prof python tools/gemm_probe.py 4096 1 > gpurun_out/ncu_gemm.log 2>&1
tail -3 gpurun_out/ncu_gemm.log
