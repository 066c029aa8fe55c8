# C5 at n = 22528 (K chunks): launch list, then one full capture of the largest emulated GEMM launch
cd $GRAFT_REPO_ROOT
python tools/c5_small.py 22528 > gpurun_out/c5_small.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python tools/c5_small.py 22528 > gpurun_out/c5_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ozaki_gemm -s 2 -c 1 -o gpurun_out/c5_ozaki python tools/c5_small.py 22528 > gpurun_out/c5_ncu2.log 2>&1
echo done; tail -2 gpurun_out/c5_ncu2.log
