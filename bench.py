#!/usr/bin/env python
"""Benchmark of the direct Monte Carlo multi-function path (BASELINE.json metric:
integrand samples/sec and seconds per 1000-function set).

Workload at N=1: BASELINE.json configs[1] = 1000 harmonic 4-D integrands
(Fig.1 family, k_n = (n+50)/2pi), 1e6 samples each, 10 trials = 1e10 samples
per step.  A step is one pass of the hot path over the whole function set.
Weak scaling: rank r integrates its own 1000 integrands (global integrand
indices r*1000 .. r*1000+999), no data-path collective.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mcb|reference]

Arms:
  mcb        device plan (descriptors resident in HBM) timed with CUDA events on
             the launching stream (`value`), plus the C-ABI call mcb_run_direct
             with host buffers timed end to end (`e2e`).
  reference  the reference's own CPU implementation (oracle/_ref, compiled from
             the unmodified reference sources; oracle port if absent) on the
             box's host cores, bounded sample of the same workload per step.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SAMPLES = 1_000_000
N_FNS = 1000
TRIALS = 10
SEED = 20200814
METRIC = "integrand samples/sec (and s per 1000-fn set) at 1/2/4/8 B200 vs CPU ref"
CONFIG_NAME = "configs[1]: 1000 harmonic 4-D integrands x 1e6 samples x 10 trials per GPU"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["mcb", "reference"], default="mcb")
    p.add_argument("--samples", type=int, default=SAMPLES)
    p.add_argument("--n-fns", type=int, default=N_FNS)
    p.add_argument("--cpu-seconds", type=float, default=12.0,
                   help="target CPU seconds for the cpu_baseline sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-clocks", action="store_true")
    p.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                   help="weak: every rank integrates its own --n-fns set (default, the driver's scaling run); "
                        "strong: the ranks split one --n-fns set")
    return p.parse_args()


# ------------------------------------------------------------------ distributed

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class Dist:
    def __init__(self, world, rank, backend):
        self.world, self.rank = world, rank
        self.backend = backend
        self.pg = None
        if world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group(backend=backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float, device=None) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=device if self.backend == "nccl" else None)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


def strong_slice(n_fns: int, rank: int, world: int):
    """Strong scaling: rank r integrates [lo, hi) of the one n_fns set."""
    return n_fns * rank // world, n_fns * (rank + 1) // world


def shard_first_index(rank: int, n_fns: int) -> int:
    """Weak scaling: rank r owns global integrand indices [r*n, (r+1)*n)."""
    return rank * n_fns


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int, enabled: bool = True):
        self.idx, self.enabled = gpu_index, enabled
        self.rows, self.proc = [], None

    def __enter__(self):
        if self.enabled:
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                     "-i", str(self.idx), "-lms", "200"], stdout=subprocess.PIPE,
                    stderr=subprocess.DEVNULL, text=True)
                self.t = threading.Thread(target=self._read, daemon=True)
                self.t.start()
            except OSError:
                self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ------------------------------------------------------------------ CPU baseline / reference arm

def cpu_reference_run(n_fns_sample: int, samples: int, first_index: int = 0):
    """The reference's run_batch (oracle/_ref) with workers=0 (all host threads),
    else the oracle port with all threads.  Returns (samples/s, seconds, kind, cores)."""
    from paper_2104_10073_b200 import workloads
    from tests import _oracle
    fns, seed, trials = workloads.c2(samples=samples, n_count=n_fns_sample, first_index=0)
    cores = os.cpu_count() or 1
    if _oracle.load_ref() is not None:
        _, _, _, _, secs = _oracle.ref_run_batch(fns, seed, trials, workers=0)
        kind = "reference"
    else:
        t0 = time.perf_counter()
        _oracle.run_direct(fns, seed, trials, n_threads=cores)
        secs = time.perf_counter() - t0
        kind = "port"
    total = n_fns_sample * samples * trials
    return total / secs, secs, kind, cores


def calibrate_cpu_sample(target_s: float, samples: int) -> int:
    rate, secs, _, _ = cpu_reference_run(max(1, os.cpu_count() or 1) // 8 or 1, samples // 10)
    per_fn = samples * TRIALS / rate
    return int(max(1, min(N_FNS, round(target_s / per_fn))))


def run_reference_arm(args, dist):
    if dist.rank != 0:
        return None
    # keep the whole arm within ~2 minutes: per-step CPU budget
    per_step = max(2.0, min(args.cpu_seconds, 100.0 / (args.steps + 0.25 * args.warmup)))
    n = calibrate_cpu_sample(per_step, args.samples)
    for _ in range(args.warmup):
        cpu_reference_run(max(1, n // 4), args.samples)
    rates, secs_all = [], []
    kind, cores = "port", os.cpu_count()
    for _ in range(args.steps):
        rate, secs, kind, cores = cpu_reference_run(n, args.samples)
        rates.append(rate)
        secs_all.append(secs)
    total_samples = n * args.samples * TRIALS * args.steps
    value = total_samples / sum(secs_all)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(secs_all) / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": CONFIG_NAME, "sample_per_step": f"{n} of {N_FNS} integrands x "
                   f"{args.samples:.0e} samples x {TRIALS} trials", "seconds_per_1000_fn_set":
                   N_FNS * args.samples * TRIALS / value},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": kind,
                         "sample": f"{n} integrands x {args.samples} samples x {TRIALS} trials per step"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    return line


# ------------------------------------------------------------------ GPU arm

def run_mcb_arm(args, dist, local):
    import numpy as np
    import torch

    import paper_2104_10073_b200 as mcb
    from paper_2104_10073_b200 import workloads

    # MCB_BENCH_SHARE_GPU=1 (test hook, gloo): ranks share the visible GPUs so the N > 1 code
    # path can run on a one-GPU box; the ranks then compete for one GPU and the numbers mean nothing
    dev = local % torch.cuda.device_count() if os.environ.get("MCB_BENCH_SHARE_GPU") == "1" else local
    torch.cuda.set_device(dev)
    if args.scaling == "strong":  # one C2 set, rank r integrates its contiguous slice
        fns, seed, trials = workloads.c2(samples=args.samples, n_count=args.n_fns)
        lo, hi = strong_slice(args.n_fns, dist.rank, dist.world)
        fns = fns[lo:hi]
    else:
        first = shard_first_index(dist.rank, args.n_fns)
        fns, seed, trials = workloads.c2(samples=args.samples, n_count=args.n_fns, first_index=first)
    arr = mcb.as_array(fns)
    stream = torch.cuda.current_stream()
    plan = mcb.Plan(arr, seed, trials, device=dev)
    info = plan.info()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{dev}")  # > 126 MB L2

    for _ in range(args.warmup):
        plan.launch(stream.cuda_stream)
    torch.cuda.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev, enabled=not args.no_clocks) as clk:
        w0 = time.perf_counter()
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the events)
            starts[i].record(stream)
            plan.launch(stream.cuda_stream)
            ends[i].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
    dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    kernel_s = sum(step_ms) * 1e-3
    kernel_s_max = dist.max(kernel_s, device=f"cuda:{dev}")
    res = plan.download(stream.cuda_stream)
    plan.close()

    # e2e: the reference-facing C-ABI call with HOST buffers (descriptor H2D,
    # kernels, result D2H inside the timed region), one call per step
    e2e_times = []
    out = None
    for i in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        out = mcb.run_direct(arr, seed, trials, devices=[dev])
        t1 = time.perf_counter()
        if i >= args.warmup:
            e2e_times.append(t1 - t0)
    e2e_s = dist.max(sum(e2e_times), device=f"cuda:{dev}")
    assert out.tobytes() == res.tobytes(), "plan and C-ABI results differ"

    job_samples = args.samples * trials * (args.n_fns if args.scaling == "strong" else args.n_fns * dist.world)
    total_samples = job_samples * args.steps
    value = total_samples / kernel_s_max
    e2e_value = total_samples / e2e_s

    # roofline of the dominant kernel (k_direct; k_combine is ~8 us of ~55 ms):
    # Philox4x32-10 blocks generated per second vs the Philox-only ceiling of
    # this GPU, measured live by the same generator code with no integrand.
    # The ceiling is set by the FP64 pipe, which on B200 executes both the
    # IMAD.WIDE multiplies of Philox and the integrand's FP64 operations
    # (tools/micro/mul_micro.cu), so frac is the share of that pipe left to
    # the sampler after the family evaluation and the reduction.
    blocks_per_launch = info.philox_blocks
    achieved = blocks_per_launch / (kernel_s / args.steps)
    peak = mcb.probe_philox_peak(dev, 50.0)
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": dist.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * kernel_s_max / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": CONFIG_NAME,
                   "integrands_per_gpu": args.n_fns if args.scaling == "weak" else len(fns),
                   "samples_per_integrand": args.samples, "trials": trials, "seed": seed,
                   "family": "cos(k*(x1+x2+x3+x4)) + sin(k*(x1+x2+x3+x4)), k_n=(n+50)/2pi, [0,1]^4",
                   "parallelism": f"{args.scaling} dp{dist.world} (integrand shards, no collective)",
                   "l2": "flushed (256 MB write) between timed iterations; inputs are ~230 KB of descriptors",
                   "seconds_per_1000_fn_set": 1e-3 * (1e3 * kernel_s_max / args.steps) * 1000 / args.n_fns,
                   "tiles_per_step": info.n_tiles, "wall_s_timed_region": wall},
        "e2e": {"value": e2e_value, "unit": "samples/s",
                "h2d_bytes_per_step": ctypes_sizeof_integrand() * len(fns),
                "d2h_bytes_per_step": int(res.nbytes),
                "path": "mcb_run_direct (C-ABI, host buffers; plan build + H2D + kernels + D2H)",
                "seconds_per_1000_fn_set": e2e_s / args.steps * 1000 / args.n_fns},
        "gpu_launches": int(info.launches_per_run) * args.steps,
        "roofline": {"bound": "alu: FP64 pipe (Philox IMAD.WIDE + integrand FP64)",
                     "achieved": achieved / 1e9, "peak": peak / 1e9, "unit": "G Philox blocks/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(),
                     "traffic_unit": "DRAM bytes per launch",
                     "blocks_per_launch": blocks_per_launch,
                     "note": "achieved = Philox4x32-10 blocks per launch (2 per 4-D sample) / k_direct "
                             "time; peak = mcb_probe_philox_peak (Philox-only, same code, measured live); "
                             "traffic = dram__bytes_read+write of this k_direct launch from " + NCU_SUMMARY +
                             " (tile table + descriptors; the kernel is ALU-bound, SURVEY.md §8(d))",
                     "hbm": hbm_roofline(ncu_traffic(), kernel_s / args.steps),
                     "fused": fused_roofline(achieved, clk.summary())},
        "clocks": clk.summary(),
    }
    return line


# Philox4x32-10 + the 14-op table harmonic on the shared IMAD.WIDE/FP64 pipe,
# blocks per clock per SM (tools/micro/split_micro.cu "ph+trig WIDE x17",
# profiles/r01_microbench.txt): the ceiling of this integrand, not of Philox alone.
FUSED_BLOCKS_PER_CLK_SM = 1.306


def fused_roofline(achieved_blocks_s, clocks):
    """The same launch against the synthetic Philox + table-trig ceiling at the
    SM clock sampled during the timed region (148 SMs)."""
    mhz = (clocks or {}).get("sm_mhz") or (clocks or {}).get("sm_max_mhz")
    if not mhz:
        return None
    peak = FUSED_BLOCKS_PER_CLK_SM * 148 * mhz * 1e6
    return {"bound": "alu: Philox + 14-op harmonic, shared IMAD.WIDE/FP64 pipe", "achieved": achieved_blocks_s / 1e9,
            "peak": peak / 1e9, "unit": "G Philox blocks/s", "frac": achieved_blocks_s / peak,
            "peak_source": "tools/micro/split_micro.cu (1.306 blocks/clk/SM) x 148 SMs x sampled SM clock"}


NCU_SUMMARY = "profiles/r01_bench_k_direct_ncu_summary.txt"


def hbm_roofline(traffic_bytes, launch_s):
    """The HBM roofline of the same launch, for reference: measured DRAM bytes
    over the launch time against MEASURED_PEAKS.json's copy bandwidth (the
    schema's "hbm" bound; ~1e-6 here — the kernel is compute-bound)."""
    if traffic_bytes is None or launch_s <= 0:
        return None
    peak = None
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as fh:
            peak = float(json.load(fh)["hbm_gbs"])
        source = "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        peak, source = 7700.0, "B200_PROFILING.md nominal"
    achieved = traffic_bytes / launch_s / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic_bytes, "peak_source": source}


def ncu_traffic():
    """DRAM bytes (read + write) of one k_direct launch of this bench's
    workload, from the committed `ncu --set full` summary (None if absent)."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), NCU_SUMMARY)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    total, found = 0.0, 0
    try:
        with open(path) as fh:
            for line in fh:
                if "DRAM read (bytes)" in line or "DRAM write (bytes)" in line:
                    parts = line.split()
                    total += float(parts[3]) * scale.get(parts[4] if len(parts) > 4 else "byte", 1)
                    found += 1
    except OSError:
        return None
    return total if found == 2 else None


def ctypes_sizeof_integrand():
    import ctypes

    import paper_2104_10073_b200 as mcb
    return ctypes.sizeof(mcb.Integrand)


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        dist = Dist(world, rank, "gloo")
        line = run_reference_arm(args, dist)
        dist.close()
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    import torch
    backend = "nccl" if torch.cuda.is_available() and os.environ.get("MCB_BENCH_SHARE_GPU") != "1" else "gloo"
    dist = Dist(world, rank, backend)
    line = run_mcb_arm(args, dist, local)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n = calibrate_cpu_sample(args.cpu_seconds, args.samples)
        rate, secs, kind, cores = cpu_reference_run(n, args.samples)
        line["cpu_baseline"] = {"value": rate, "unit": "samples/s", "cores": cores, "kind": kind,
                                "sample": f"{n} of {N_FNS} integrands x {args.samples} samples x "
                                          f"{TRIALS} trials ({secs:.1f} s)"}
    dist.close()
    if rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
