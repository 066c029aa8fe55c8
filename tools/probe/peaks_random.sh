# INT8 tensor-core probes with clock + power recorded per leg:
#  (1) issue-rate probe, constant operands (burst peak, as in peaks.sh)
#  (2) the same MMA stream on uniformly random int8 digits rotated MMA to MMA,
#      back to back for ~4 s (what the power cap sustains on real digit data)
#  (3) the library INT8 GEMM (torch._int_mm -> cuBLASLt) 16384^3, burst and sustained
cd $GRAFT_REPO_ROOT
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17"
$NV tools/probe/i8_peak.cu -o tools/probe/i8_peak.bin || exit 1
leg() {  # name, command...
  name=$1; shift
  nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 100 > gpurun_out/peak_clocks_$name.csv &
  SMI=$!
  sleep 0.5
  echo "== $name"; "$@"
  kill $SMI; wait $SMI 2>/dev/null
  python - "$name" <<'PY'
import csv, statistics, sys
rows=[r for r in csv.reader(open(f'gpurun_out/peak_clocks_{sys.argv[1]}.csv')) if len(r) >= 5]
busy=[(float(r[1].split()[0]), float(r[3].split()[0]), r[4].strip()) for r in rows if float(r[3].split()[0]) > 300]
if busy:
    print("   clocks under load: sm_mhz median", statistics.median(s for s,_,_ in busy), "min", min(s for s,_,_ in busy),
          "| power W median", statistics.median(p for _,p,_ in busy), "max", max(p for _,p,_ in busy),
          "| sw_power_cap active in", sum(1 for *_,c in busy if c == 'Active'), "of", len(busy), "samples")
PY
}
med() { awk '{for(i=1;i<=NF;i++) if ($i=="TOPS") print $(i-1)}' | sort -n | awk '{a[NR]=$1} END {print "   TOPS min", a[1], "median", a[int((NR+1)/2)], "max", a[NR], "(" NR " launches)"}'; }
leg const_sustained bash -c './tools/probe/i8_peak.bin sustained' | { tee /dev/stderr | grep TOPS | med; } 2>&1 | grep -v "^N="
leg random_sustained bash -c './tools/probe/i8_peak.bin random' | { tee /dev/stderr | grep TOPS | med; } 2>&1 | grep -v "^N="
leg int_mm python - <<'PY'
import torch, time
n = 16384
a = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 128, (n, n), dtype=torch.int8, device="cuda")
try:
    for _ in range(3): torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); torch._int_mm(a, b); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"   torch._int_mm {n}^3 burst (best of 10): {best:.3f} ms, {2*n**3/best/1e9:.1f} TOPS")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = 0; t0 = time.time(); e0.record()
    while time.time() - t0 < 4.0:
        for _ in range(10): torch._int_mm(a, b)
        k += 10; torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    print(f"   torch._int_mm {n}^3 sustained (4 s back to back): {ms:.3f} ms, {2*n**3/ms/1e9:.1f} TOPS")
except Exception as ex:
    print("   torch._int_mm unavailable:", repr(ex)[:200])
PY
