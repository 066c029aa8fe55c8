# K-chunked emulated GEMM parity test (C5 chain at n = 22528 > 21000)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "k_chunks or emulated" --durations=5 > gpurun_out/kchunk_test.log 2>&1; echo "test rc=$?" >> gpurun_out/kchunk_test.log
tail -12 gpurun_out/kchunk_test.log
