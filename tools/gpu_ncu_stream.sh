cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:stream_reduce_all_pairs_block -c 2 -o gpurun_out/r02_C3_stream python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-strict > gpurun_out/ncu_stream.log 2>&1; echo "rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:stream_reduce_warp_pairs -c 1 -o gpurun_out/r02_C3_stream_warp python bench.py --config C3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-strict > gpurun_out/ncu_stream2.log 2>&1; echo "rc=$?"
