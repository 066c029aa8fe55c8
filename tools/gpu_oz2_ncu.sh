cd $GRAFT_REPO_ROOT
for m in 1 0; do
USTATS_OZ_2SM=$m timeout 600 ncu --set full --clock-control none -k regex:ozaki_gemm -c 1 -o gpurun_out/oz_sym_$m python tools/oz_one.py 8192 sym 6 > gpurun_out/ncu_oz_$m.log 2>&1
echo "ncu $m rc=$?"; tail -3 gpurun_out/ncu_oz_$m.log
done
