set -x
nvidia-smi; nproc; lscpu | grep -E 'Model name|Socket|Core|Thread'; free -g
./tools/probe/dmma_peak
python - <<'PY'
import torch, time
for n in (4096, 8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device='cuda'); b = torch.randn(n, n, dtype=torch.float64, device='cuda')
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(f"cuBLAS DGEMM n={n}: {2*n**3/best/1e9:.2f} TFLOP/s ({best:.2f} ms)")
    if n == 8192:
        t0=time.time(); e0.record()
        for _ in range(20): c = a @ b
        e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1)/20
        print(f"cuBLAS DGEMM n={n} sustained: {2*n**3/ms/1e9:.2f} TFLOP/s")
PY
