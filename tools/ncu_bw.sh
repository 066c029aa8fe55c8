# per-kernel DRAM throughput of the bandwidth-bound kernels (one step each)
cd $GRAFT_REPO_ROOT
for CFG in C1 C2 C4; do
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_bw_$CFG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/bw_$CFG.csv -k regex:"stream_|sweep|pair_sym|gemm_tma" $CMD > gpurun_out/ncu_bw_$CFG.log 2>&1
echo "$CFG rc=$?"
done
