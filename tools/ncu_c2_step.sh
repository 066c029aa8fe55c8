# full ncu capture of the emulated GEMM inside the C2 bench step (current build)
cd $GRAFT_REPO_ROOT
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c2_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ozaki_gemm -s 3 -c 1 -o gpurun_out/c2_ozaki_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c2_full.log 2>&1
echo "rc=$?"; tail -c 300 gpurun_out/c2_plain.json
