cd $GRAFT_REPO_ROOT
USTATS_OZ_2SM=1 timeout 180 python tools/oz2_check.py 2>&1 | tail -4
USTATS_OZ_2SM=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:ozaki_gemm -c 1 -o gpurun_out/oz_sym_1b python tools/oz_one.py 8192 sym 6 > gpurun_out/ncu_oz_1b.log 2>&1; echo "ncu rc=$?"
