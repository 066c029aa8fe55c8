# full ncu capture of the stream (bandwidth) kernels of one C2 and one C4 step
cd $GRAFT_REPO_ROOT
for CFG in C2 C4; do
CMD="python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$CFG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stream_" -c 6 -o gpurun_out/streams_$CFG $CMD > gpurun_out/ncu_streams_$CFG.log 2>&1
echo "$CFG rc=$?"
done
