cd $GRAFT_REPO_ROOT
python tools/ozaki_one.py 8192 > gpurun_out/oz_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ozaki_gemm -c 1 -o gpurun_out/ozaki_full python tools/ozaki_one.py 8192 > gpurun_out/ncu_ozaki.log 2>&1
echo "rc=$?"; cat gpurun_out/oz_plain.log
