# C5 at full size (n = 65536): launch list, then one full capture of an emulated GEMM launch
cd $GRAFT_REPO_ROOT
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_full_launches.csv python tools/run_c5.py 65536 > gpurun_out/c5_full_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ozaki_gemm -s 2 -c 1 -o gpurun_out/c5_full_ozaki python tools/run_c5.py 65536 > gpurun_out/c5_full_ncu2.log 2>&1
echo done; tail -2 gpurun_out/c5_full_ncu2.log
