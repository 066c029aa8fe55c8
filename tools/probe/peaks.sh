# Tensor-core peak probes with the SM clock recorded while they run:
# INT8 tcgen05.mma (kind::i8, M128 x N x K32, 148 CTAs) and FP64 DMMA
# (mma.sync m8n8k4), burst and sustained; cuBLAS DGEMM for reference.
cd $GRAFT_REPO_ROOT
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17"
$NV tools/probe/i8_peak.cu -o tools/probe/i8_peak.bin && $NV tools/probe/dmma_peak.cu -o tools/probe/dmma_peak.bin || exit 1
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,temperature.gpu --format=csv,noheader -lms 100 > gpurun_out/peak_clocks.csv &
SMI=$!
sleep 1
echo "== INT8 burst"; ./tools/probe/i8_peak.bin
echo "== INT8 sustained (300 launches of N=256)"; ./tools/probe/i8_peak.bin sustained | awk '{print $6}' | sort -n | awk '{a[NR]=$1} END {print "TOPS min", a[1], "median", a[int(NR/2)], "max", a[NR]}'
echo "== FP64 DMMA"; ./tools/probe/dmma_peak.bin
kill $SMI
echo "== clocks while probing (MHz, W)"; python - <<'PY'
import csv, statistics
rows=[r for r in csv.reader(open('gpurun_out/peak_clocks.csv')) if len(r) >= 5]
sm=[float(r[1].split()[0]) for r in rows]; pw=[float(r[3].split()[0]) for r in rows]
busy=[(s,p,r[4].strip()) for s,p,r in zip(sm,pw,rows) if p > 300]
print("samples", len(rows), "under load", len(busy))
if busy:
    print("sm_mhz median under load", statistics.median(s for s,_,_ in busy), "max clock", max(float(r[2].split()[0]) for r in rows))
    print("power max", max(p for _,p,_ in busy), "sw_power_cap active in", sum(1 for *_,c in busy if c == 'Active'), "samples")
PY
