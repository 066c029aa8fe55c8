# iteration loop: GPU parity tests + GEMM probe
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | grep -v "^  File" | tail -15
timeout 300 python tools/gemm_probe.py 4096 2
timeout 300 python tools/gemm_probe.py 8192 2
