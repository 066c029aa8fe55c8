# INT8 tcgen05 peak probe, C2 bench (Ozaki path), launch list, full ncu capture of the Ozaki GEMM
cd $GRAFT_REPO_ROOT
./tools/probe/i8_peak.bin > gpurun_out/int8_peak_probe.log 2>&1; cat gpurun_out/int8_peak_probe.log
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ozaki_gemm -c 1 -o gpurun_out/ozaki_c2_full $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
