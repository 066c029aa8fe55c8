#!/usr/bin/env python
"""Exact U-statistic throughput on B200 (BASELINE.json metric: evals/s and % of
the FP64 tensor-core / HBM roofline at 1/2/4/8 B200).

One step = one exact U-statistic evaluation of the workload (device
tensorization of the components from the raw sample, every sparsified
partition-lattice V-term contracted on the GPU, the per-term values combined
on the host in the reference's order). Default workload: BASELINE.json
configs[4] (C5, m=7 HOIF chain, n=65536, a 34 GB factor): the config the
metric is quoted on at 1/2/4/8 GPUs; it fits one B200 (`--config C1..C4` for
the others).

  value  sample resident in HBM (device pointer through the C-ABI)
  e2e    the same public call with the sample in pinned HOST memory: its H2D
         and the D2H of the terms inside every timed step

`--impl reference` times the reference's own CPU implementation
(oracle/_ref, compiled from /root/reference sources) on this host's cores:
full size where that finishes in the run's time budget (C1, C2; C3 with few
steps), else a bounded sample per step extrapolated to the config's n with
the reference's exact multiply-add polynomial (C4, C5: the full-size CPU run
needs ~1e6 s and >= 0.4 TB of RAM), labelled as such.

N>1 (torchrun): V-terms are LPT-sharded over ranks and shared GEMMs are split
into row panels; per-term values meet in one NCCL all-reduce.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# measured peaks with the SM clock recorded while the probes ran (1965 MHz, no
# throttle reason; tools/probe/peaks.sh -> profiles/r02_peak_probes.log)
FP64_PEAK_TFLOPS = 37.04      # mma.sync f64 m8n8k4 issue-rate probe (best configuration)
FP64_CUBLAS_TFLOPS = 36.17    # cuBLAS DGEMM 16384^3 on this pool (profiles/r01_fp64_peak_probe.log)
INT8_PEAK_TOPS = 4542.7       # tcgen05.mma kind::i8 M128 N256 K32 on 148 SMs, median of 300 back-to-back launches
PROBE_MHZ = 1965.0            # SM clock the probes ran at
# The issue-rate probe multiplies one resident tile of small constants: 390-530 W,
# no power cap. The same MMA stream on uniformly random int8 digits (what a digit
# GEMM feeds the tensor cores) rotated MMA to MMA, back to back for ~4 s, hits the
# 1000 W cap with NO data movement at all: median 1680 MHz, 3867 TOPS
# (tools/probe/peaks_random.sh -> profiles/r02_int8_sustained_probe.log). That is
# the sustained INT8 ceiling of this GPU on real data; the library INT8 GEMM
# (torch._int_mm -> cuBLASLt, 16384^3) measured beside it: 2678 TOPS burst,
# 2019 TOPS sustained (862 MHz under the cap).
INT8_SUSTAINED_TOPS = 3867.3
INT8_LIBRARY_GEMM_TOPS = {"burst": 2678.3, "sustained": 2019.4}


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                parts.append(time.time())
                self.rows.append(parts)

    def wait_ready(self, timeout: float = 5.0):
        """nvidia-smi's start-up (NVML init) perturbs the GPU: start the sampler
        before the warm-up and wait for its first sample."""
        t0 = time.time()
        while self.proc and not self.rows and time.time() - t0 < timeout:
            time.sleep(0.05)

    def mark(self, start: float, end: float):
        self.window = (start, end)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        rows = self.rows
        win = getattr(self, "window", None)
        if win:
            inside = [r for r in rows if win[0] - 0.25 <= r[-1] <= win[1] + 0.25]
            rows = inside or rows[-2:]  # short regions: the samples bracketing them
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if str(r[4 + i]).lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def reference_sample(name: str, n_sample: int, threads: int, repeats: int = 1, data_api: bool = True):
    """Times the reference u_statistic (oracle/_ref) on a bounded sample: with
    data_api, the reference's own call on the raw sample (its tensorize
    evaluates the RBF / projection components per entry); otherwise on
    pre-tensorized factors."""
    from oracle import ref as REF
    from paper_2508_12627_b200.workloads import generate, generate_data
    cap = max(2 ** 31, n_sample ** 3 + 1)
    walls, stats = [], None
    if data_api:
        data, spec, m, _ = generate_data(name, n_sample)
        for _ in range(repeats):
            t0 = time.perf_counter()
            u, stats = REF.u_statistic_data(spec, data, threads=threads, cap=cap)
            walls.append(time.perf_counter() - t0)
        return u, min(walls), stats
    factors, sig, m, _ = generate(name, n_sample)
    for _ in range(repeats):
        t0 = time.perf_counter()
        u, stats = REF.u_statistic(factors, sig, m, threads=threads, cap=cap)
        walls.append(time.perf_counter() - t0)
    return u, min(walls), stats


# Bounded reference sample per config: C1 and C2 run at full size; C3's full
# size (~10 min per evaluation) only when the run's step count fits the budget;
# C4 and C5 are infeasible at full size on any host (C4 ~1.5 h and ~300 GB of
# concurrent n^3 buffers, C5 ~1e6 s and >= 0.4 TB), so they are timed at the
# sample n and extrapolated with the reference's EXACT multiply-add polynomial
# (C5 241 n^3 + 1534 n^2 + ..., C4 51 n^4 + ...).
CPU_SAMPLE_N = {"C1": 2000, "C2": 4096, "C3": 4096, "C4": 192, "C5": 2048}
FULL_FEASIBLE = {"C1", "C2", "C3"}
REFERENCE_ARM_BUDGET_S = 1500.0
_MADDS = {}


def reference_madds(name, n):
    """Exact reference-plan multiply-adds (ExecStats rules, einsum.cpp) at extent
    n: the polynomial of degree <= m fitted EXACTLY (integer coefficients) to
    the reference's own counts at small n."""
    from paper_2508_12627_b200.workloads import CONFIGS
    from oracle import ref as REF
    w = CONFIGS[name]
    if name not in _MADDS:
        sig = [list(t) for t in w.signature]
        xs = list(range(w.m + 2, 2 * w.m + 5))
        ys = []
        for x in xs:
            rng = np.random.default_rng(0)
            facs = [rng.uniform(0.5, 1.5, size=(x,) * len(t)) for t in sig]
            _, st = REF.u_statistic(facs, sig, w.m, threads=1)
            ys.append(st["multiply_adds"])
        _MADDS[name] = np.round(np.polyfit(np.array(xs, float), np.array(ys, float), w.m))
    return float(np.polyval(_MADDS[name], float(n)))


def extrapolated_seconds(name, n, n_s, wall, stats):
    """Reference time at n from a run at n_s: tensorize ~ n^2 (one callback per
    entry per component), contraction ~ the exact multiply-add polynomial, the
    rest (enumeration, planning) as measured."""
    tz, tc = stats["tensorize_seconds"], stats["contract_seconds"]
    rest = max(0.0, wall - tz - tc)
    return tz * (n / n_s) ** 2 + tc * reference_madds(name, n) / reference_madds(name, n_s) + rest


def reference_plan(name, n, threads, data_api, runs):
    """Decides full size vs bounded sample for `runs` reference evaluations.
    Returns (run_n, full, detail)."""
    n_s = min(CPU_SAMPLE_N[name], n)
    if n_s == n:
        return n, True, {}
    if name not in FULL_FEASIBLE:
        return n_s, False, {}
    _, t_s, st = reference_sample(name, n_s, threads, data_api=data_api)  # one probe predicts full size
    est = extrapolated_seconds(name, n, n_s, t_s, st)
    full = est * runs <= REFERENCE_ARM_BUDGET_S
    return (n if full else n_s), full, {"probe_n": n_s, "probe_wall": t_s, "full_estimate_s": est}


def run_reference_arm(args, name, world, rank):
    if rank != 0:
        return 0
    from oracle import ref as REF
    if not REF.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libustats_ref.so not built"}))
        return 0
    from paper_2508_12627_b200.workloads import CONFIGS
    w = CONFIGS[name]
    n = args.n or w.n
    threads = os.cpu_count() or 1
    data_api = args.api == "data"
    run_n, full, det = reference_plan(name, n, threads, data_api, args.steps + args.warmup)
    for _ in range(args.warmup):
        reference_sample(name, run_n, threads, data_api=data_api)
    secs, walls = [], []
    for _ in range(args.steps):
        _, wall, st = reference_sample(name, run_n, threads, data_api=data_api)
        walls.append(wall)
        secs.append(wall if full else extrapolated_seconds(name, n, run_n, wall, st))
    t_full = statistics.mean(secs)
    call = "u_statistic(kernel spec, sample) incl. its tensorize" if data_api else "u_statistic on tensor-backed components"
    if full:
        sample = (f"ustats::u_statistic (oracle/_ref: the unmodified reference sources), {call}, at FULL n={n}, "
                  f"threads={threads}, mean wall {t_full:.3f}s over {len(secs)} runs")
    else:
        sample = (f"EXTRAPOLATED: ustats::u_statistic (oracle/_ref), {call}, at n={run_n}, threads={threads}, "
                  f"mean wall {statistics.mean(walls):.3f}s over {len(walls)} runs; each run scaled to n={n} "
                  f"(tensorize x (n/{run_n})^2, contraction x madds({n})/madds({run_n}) = "
                  f"{reference_madds(name, n):.4g}/{reference_madds(name, run_n):.4g}, the reference's exact "
                  f"multiply-add polynomial)")
    value = 1.0 / t_full
    line = {
        "metric": "U-statistic exact evals/sec", "value": value, "unit": "evals/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_full * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json construction)",
        "config": {"workload": name, "m": w.m, "n": n, "signature": [list(t) for t in w.signature]},
        "same_config": bool(full), "sample_n": run_n,
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "reference", "sample": sample,
                         "extrapolated": not full},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if det:
        line["probe"] = det
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--n", type=int, default=0, help="override the config's n (parity/debug only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-strict", action="store_true", help="skip the FP64-strict (DMMA-only) roofline leg")
    ap.add_argument("--budget-s", type=float, default=1400.0,
                    help="wall budget of the whole run: the e2e and FP64-strict legs shrink to fit it")
    ap.add_argument("--api", default="data", choices=["data", "tensors"],
                    help="data: u_statistic(spec, sample) with GPU tensorization (the binding's call); "
                         "tensors: pre-tensorized factors (us_u_terms)")
    ap.add_argument("--shard", default="rows", choices=["rows", "terms"],
                    help="N>1: row-shard every op (NCCL inside the engine) or shard V-terms")
    args = ap.parse_args()
    world, rank, local = dist_env()
    name = args.config
    t_begin = time.time()

    if args.impl == "reference":
        return run_reference_arm(args, name, world, rank)

    import torch
    import paper_2508_12627_b200 as us
    from paper_2508_12627_b200.workloads import CONFIGS, generate, input_bytes

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if args.shard == "rows":
            from paper_2508_12627_b200.distributed import init_row_sharding
            init_row_sharding(local)
    w = CONFIGS[name]
    n = args.n or w.n
    use_data = args.api == "data" and not (world > 1 and args.shard == "terms")
    cfg = us.Config(device=local, rank=rank, world_size=world, shard_rows=(world > 1 and args.shard == "rows"),
                    memory_cap_entries=max(2 ** 31, n * n + 1, n ** 3 + 1 if name == "C4" else 0))
    # the reference needs memory_cap_entries raised past n^2 for C5 (tensor.cpp:9-23);
    # SURVEY 8d prescribes the same for its CPU baseline
    if use_data:
        # the binding's public call: u_statistic(kernel spec, sample); the
        # components are tensorized on the GPU from the sample
        from paper_2508_12627_b200.workloads import generate_data
        data, spec, m, _ = generate_data(name, n)
        sig = [list(t) for t in w.signature]
        dX = torch.from_numpy(data).cuda()
        hX = torch.from_numpy(data).pin_memory()
        dfac, hfac = dX, hX
        in_bytes = data.nbytes
    else:
        factors, sig, m, _ = generate(name, n)
        spec = None
        # device-resident and pinned-host copies (aliases preserved)
        dev, pin, dfac, hfac = {}, {}, [], []
        for f in factors:
            if id(f) not in dev:
                t = torch.from_numpy(f)
                dev[id(f)] = t.cuda()
                pin[id(f)] = t.pin_memory()
            dfac.append(dev[id(f)])
            hfac.append(pin[id(f)])
        in_bytes = input_bytes(factors)
    torch.cuda.synchronize()

    class _R:  # per-step result: value + engine stats
        def __init__(self, value, stats, terms):
            self.value, self.stats, self.terms = value, stats, terms

    def step(fx, on_device):
        if use_data:
            u, st = us.u_statistic(spec, fx, config=cfg, with_stats=True)
            return u, _R(u, st, int(st["partitions_evaluated"]))
        r = us.u_terms(fx, sig, m, cfg) if on_device else _host_terms(us, fx, sig, m, cfg)
        if world > 1 and not cfg.shard_rows:  # term sharding: one all-reduce of the V vector
            import torch.distributed as dist
            v = torch.from_numpy(r.v).cuda()
            dist.all_reduce(v)
            u = us.combine_terms(r.mu, v.cpu().numpy())
        else:
            u = r.value
        return u, _R(u, r.stats, len(r.v))

    # Inputs smaller than L2 (126 MB) would stay cached across steps: flush L2
    # between steps (write a 512 MiB buffer) and time each step on its own.
    flush = in_bytes < 126e6
    scrub = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda") if flush else None

    def timed(fx, on_device, k):
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        last = None
        if flush:
            ms = 0.0
            for _ in range(k):
                scrub.fill_(1.0)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                last = step(fx, on_device)
                e1.record()
                torch.cuda.synchronize()
                ms += e0.elapsed_time(e1)
                if os.environ.get("BENCH_STEP_TIMES"):
                    print(f"step {e0.elapsed_time(e1):.3f} ms", file=sys.stderr)
        else:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(k):
                last = step(fx, on_device)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms / k, last

    # Repeated small data-API evaluations (n <= 4096) replay one captured CUDA
    # graph; the engine's per-class event records would switch that off, so for
    # those configs the kernel-class times come from a separate profiled pass
    # right after the timed region (same inputs, same build), not from inside it.
    separate_profile = use_data and world == 1 and n <= 4096
    with ClockSampler(local) as clocks:
        clocks.wait_ready()
        for _ in range(args.warmup):
            step(dfac, True)
        if not separate_profile:
            us.profile(enable=True, reset=True, device=local)
        replays0 = us.graph_replays(local)
        t_start = time.time()
        ms_step, (u_val, r) = timed(dfac, True, args.steps)
        clocks.mark(t_start, time.time())
        replayed = us.graph_replays(local) - replays0
        if separate_profile:
            us.profile(enable=True, reset=True, device=local)
            for _ in range(args.steps):
                _, r = step(dfac, True)
            torch.cuda.synchronize()
        prof = us.profile(enable=False, reset=True, device=local)
    e2e = None
    step_s = ms_step * 1e-3
    strict_s = 3.5 * step_s if (cfg.fp64_emulation and not args.no_strict) else 0.0  # DMMA ~3x slower
    if not args.no_e2e:
        # e2e repeats the timed loop with host buffers; a long step (C5) runs
        # fewer e2e steps so the whole bench stays inside --budget-s
        left = args.budget_s - (time.time() - t_begin) - strict_s
        e2e_steps = args.steps if left >= (args.steps + 1) * step_s else max(3, min(args.steps, int(left / step_s) - 1))
        if step_s > 5.0:  # a long step (C5): three e2e evaluations measure it; the run stays within minutes
            e2e_steps = min(e2e_steps, 3)
        if step_s < 5.0:
            # warm the host-buffer path as the device path was warmed (pinned registration, the plan,
            # and for small problems the one-off graph capture); a long step needs none
            for _ in range(min(3, max(1, args.warmup))):
                step(hfac, False)
        e2e_ms, _ = timed(hfac, False, e2e_steps)
        e2e = {"value": 1e3 / e2e_ms, "unit": "evals/s", "h2d_bytes_per_step": int(in_bytes),
               "d2h_bytes_per_step": 8 * int(r.terms) + (4 if use_data else 0), "ms_per_step": e2e_ms,
               "steps": e2e_steps,
               "call": f"u_statistic('{spec}', pinned host sample)" if use_data else "us_u_terms(host tensors)"}
    strict = None
    if strict_s > 0 and world == 1 and time.time() - t_begin + strict_s < args.budget_s:
        # FP64-strict leg: the same evaluation with every GEMM on the FP64 DMMA
        # tensor cores (no INT8 emulation) -> the IEEE-FP64 roofline beside the emulated one
        import dataclasses
        scfg = dataclasses.replace(cfg, fp64_emulation=False)

        def sstep():
            if use_data:
                return us.u_statistic(spec, dfac, config=scfg, with_stats=True)
            rr = us.u_terms(dfac, sig, m, scfg)
            return rr.value, rr.stats
        nst = 1 if strict_s > 30 else max(1, min(args.steps, int(30 / max(strict_s, 1e-3))))
        if strict_s <= 30:
            sstep()  # plan + warm
        us.profile(enable=True, reset=True, device=local)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(nst):
            su, sst = sstep()
        torch.cuda.synchronize()
        s_wall = (time.perf_counter() - t0) / nst
        sprof = us.profile(enable=False, reset=True, device=local)
        s_gemm_ms = sprof["gemm_ms"] / nst
        s_ach = 2.0 * sst["executed_gemm_macs"] / (s_gemm_ms * 1e-3) / 1e12 if s_gemm_ms > 0 else None
        strict = {"value": 1.0 / s_wall, "unit": "evals/s", "steps": nst, "u": su,
                  "u_minus_emulated_u": su - u_val,
                  "roofline": {"bound": "tensor", "achieved": s_ach, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                               "frac": s_ach / FP64_PEAK_TFLOPS if s_ach else None,
                               "kernel": "gemm_tma_kernel (TMA + DMMA.8x8x4, FP64 tensor pipe)",
                               "kernel_ms_per_step": s_gemm_ms, "kernel_share_of_step": s_gemm_ms / (s_wall * 1e3)},
                  "timing": "host wall per evaluation (plan cached when steps > 1), GEMM time from CUDA events"}

    st = r.stats
    gemm_ms = prof["gemm_ms"] / args.steps
    stream_ms = prof["stream_ms"] / args.steps
    peaks = measured_peaks()
    if st.get("int8_tensor_ops", 0) > 0 and st.get("emulated_gemm_macs", 0) * 2 > st["executed_gemm_macs"]:
        # FP64 GEMMs emulated on the INT8 tensor cores (Ozaki digits): the
        # dominant kernel's roofline is the INT8 tcgen05 rate
        achieved = st["int8_tensor_ops"] / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
        roofline = {"bound": "tensor", "achieved": achieved, "peak": INT8_PEAK_TOPS, "unit": "TOPS (int8)",
                    "frac": achieved / INT8_PEAK_TOPS if achieved else None,
                    "kernel": "ozaki_gemm_kernel (tcgen05.mma kind::i8, TMEM accumulators) + digit split + epilogue pass",
                    "kernel_ms_per_step": gemm_ms, "kernel_share_of_step": gemm_ms / ms_step,
                    "fp64_equivalent_tflops": 2.0 * st["executed_gemm_macs"] / (gemm_ms * 1e-3) / 1e12
                    if gemm_ms > 0 else None,
                    "fp64_dmma_peak_tflops": FP64_PEAK_TFLOPS,
                    "peak_source": f"burst: measured INT8 tcgen05 issue-rate probe {INT8_PEAK_TOPS} TOPS (M128 N256 K32, "
                                   f"148 SMs, constant operands, 1965 MHz, 530 W, profiles/r02_peak_probes.log); "
                                   f"MEASURED_PEAKS.json has no INT8 entry",
                    "peak_sustained": INT8_SUSTAINED_TOPS,
                    "frac_sustained": achieved / INT8_SUSTAINED_TOPS if achieved else None,
                    "peak_sustained_source": "the same probe on random int8 digits rotated MMA to MMA for 4 s: power-capped "
                                             "(1000 W) at 1680 MHz with no data movement "
                                             "(profiles/r02_int8_sustained_probe.log)",
                    "library_int8_gemm_tops": INT8_LIBRARY_GEMM_TOPS,
                    "traffic": ncu_traffic(name, "gemm")}
    elif st["executed_gemm_macs"] > 0:
        achieved = 2.0 * st["executed_gemm_macs"] / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
        roofline = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                    "frac": achieved / FP64_PEAK_TFLOPS if achieved else None,
                    "kernel": "gemm_tma_kernel (TMA + DMMA.8x8x4)", "kernel_ms_per_step": gemm_ms,
                    "kernel_share_of_step": gemm_ms / ms_step,
                    "peak_source": f"measured FP64 DMMA issue-rate probe {FP64_PEAK_TFLOPS} TFLOP/s "
                                   f"(cuBLAS DGEMM {FP64_CUBLAS_TFLOPS}); MEASURED_PEAKS.json has no FP64 entry",
                    "traffic": ncu_traffic(name, "gemm")}
    else:
        bytes_step = 8.0 * st["executed_stream_entries"]
        achieved = bytes_step / (stream_ms * 1e-3) / 1e9 if stream_ms > 0 else None
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                    "frac": achieved / peaks["hbm_gbs"] if achieved else None,
                    "kernel": "stream kernels", "kernel_ms_per_step": stream_ms,
                    "kernel_share_of_step": stream_ms / ms_step, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                    "traffic": ncu_traffic(name, "stream")}
    clk = clocks.summary()
    if roofline.get("bound") == "tensor" and roofline.get("achieved") and clk.get("sm_mhz"):
        # the probe peaks were measured at 1965 MHz; a power-capped run's tensor
        # pipes run at the sampled median clock (sw_power_cap): the fraction of
        # the peak at that clock says how busy the kernel keeps them
        roofline["frac_at_sampled_clock"] = roofline["achieved"] / (roofline["peak"] * clk["sm_mhz"] / PROBE_MHZ)
    line = {
        "metric": "U-statistic exact evals/sec", "value": 1e3 / ms_step * 1, "unit": "evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json construction)",
        "config": {"workload": name, "m": m, "n": n, "signature": sig, "terms": int(r.terms),
                   "api": (f"u_statistic('{spec}', sample): components tensorized on the GPU"
                           if use_data else "u_terms(tensors)"),
                   "gemm": ("FP64 via Ozaki splitting on the INT8 tensor cores (S balanced 8-bit digits per value, S "
                            "from the error-bound guard: worst-case entry error <= that of the FP64 dot product, S=6 "
                            "for K >= 1024; exact int32 digit products, FP64 assembly) where K >= 1024 (long K in "
                            "chunks summed in FP64; consumers of C^2 then stay on DMMA), else FP64 DMMA")
                   if cfg.fp64_emulation else "FP64 DMMA (mma.sync f64)",
                   "parallelism": (f"row-sharded x{world}" if args.shard == "rows" else f"term-sharded x{world}")
                   if world > 1 else "single GPU",
                   "l2": "inputs larger than L2 (no flush needed)" if not flush
                   else "L2 flushed (512 MiB write) before every timed step; steps timed individually"},
        "u": u_val,
        "roofline": roofline,
        "gpu_launches": int(st["kernel_launches"]) * args.steps,
        "clocks": clk,
        "stats_per_step": {k: st[k] for k in ("multiply_adds", "executed_gemm_macs", "executed_stream_entries",
                                               "gemm_launches", "stream_launches", "shared_hits",
                                               "emulated_gemm_macs", "int8_tensor_ops", "oz_slices")},
        "stream_ms_per_step": stream_ms,
        "graph_replayed_steps": int(replayed),
        "kernel_times_from": ("a separate profiled pass of the same steps (event records inside the timed region "
                              "would disable the CUDA-graph replay)") if separate_profile else "the timed region",
    }
    if e2e:
        line["e2e"] = e2e
    if strict:
        line["fp64_strict"] = strict
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(name, n, use_data)
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def _host_terms(us, fx, sig, m, cfg):
    # pinned host tensors -> host pointers (on_device=0): the engine's own H2D
    import ctypes as C
    from paper_2508_12627_b200 import _native as N
    from paper_2508_12627_b200.api import UTerms, _check, _signature
    K, L, I = _signature(sig)
    seen, ptrs = {}, []
    for t in fx:
        ptrs.append(t.data_ptr())
    P = (C.c_void_p * K)(*ptrs)
    n = fx[1].shape[0] if fx[1].dim() else fx[0].shape[0]
    cap = us.bell_number(m)
    rgs = np.zeros((cap, m), dtype=np.int32)
    mu = np.zeros(cap, dtype=np.int64)
    v = np.zeros(cap)
    own = np.zeros(cap, dtype=np.int32)
    cnt, u = N.i32(), N.f64()
    st = N.UsStats()
    c = cfg.native()
    _check(N.lib().us_u_terms(m, K, L, I, P, n, 0, C.byref(c), cap, C.byref(cnt),
                              rgs.ctypes.data_as(C.POINTER(N.i32)), mu.ctypes.data_as(C.POINTER(N.i64)),
                              v.ctypes.data_as(C.POINTER(N.f64)), own.ctypes.data_as(C.POINTER(N.i32)),
                              C.byref(u), C.byref(st)))
    T = cnt.value
    return UTerms(u.value, rgs[:T], mu[:T], v[:T], own[:T], st.as_dict())


def ncu_traffic(name, kind):
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text())
    entry = d.get(name, {}).get(kind)
    return entry.get("bytes_per_launch") if isinstance(entry, dict) else entry


def cpu_baseline(name, n, data_api=True):
    """The reference CPU path on this host, one bounded run (rank 0, N=1): full
    size for C1, else the config's sample n extrapolated with the exact
    multiply-add polynomial (as in the reference arm)."""
    from oracle import ref as REF
    if not REF.available():
        return {"value": None, "unit": "evals/s", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built on this host"}
    threads = os.cpu_count() or 1
    n_s = min(CPU_SAMPLE_N[name], n)
    _, wall, st = reference_sample(name, n_s, threads, data_api=data_api)
    if n_s == n:
        return {"value": 1.0 / wall, "unit": "evals/s", "cores": threads, "kind": "reference", "extrapolated": False,
                "sample": f"ustats::u_statistic (oracle/_ref) at full n={n}, threads={threads}: {wall:.3f}s wall"}
    est = extrapolated_seconds(name, n, n_s, wall, st)
    return {"value": 1.0 / est, "unit": "evals/s", "cores": threads, "kind": "reference", "extrapolated": True,
            "sample": (f"ustats::u_statistic (unmodified reference, oracle/_ref) on the "
                       f"{'raw sample (its tensorize included)' if data_api else 'tensorized factors'}, "
                       f"threads={threads}: {wall:.3f}s at n={n_s} (tensorize {st['tensorize_seconds']:.3f}s, "
                       f"contract {st['contract_seconds']:.3f}s), extrapolated to n={n} with the exact "
                       f"multiply-add polynomial (contract) and n^2 (tensorize): {est:.4g}s")}


if __name__ == "__main__":
    sys.exit(main())
