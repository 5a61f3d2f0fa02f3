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
             with host buffers timed end to end (`e2e`; at N > 1 rank 0 calls it
             with every GPU in the device list, so the product's own multi-GPU
             scheduler is what is timed).  At N = 1 the line also carries the
             other BASELINE configs (`configs`: C1, C3, C4, C5 device-timed) and,
             at N > 1, configs[4] (C5) weak and strong (`scaling_c5`).
  reference  the reference's own CPU implementation (oracle/_ref: its run_batch
             compiled from the unmodified sources, reached through the extern "C"
             shim; the oracle port only if that library is absent) on the box's
             host cores, a strided sample of the same workload per step.  This
             arm never imports the paper_2104_10073_b200 package.
"""
from __future__ import annotations

import argparse
import ctypes
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
FAMILY = "cos(k*(x1+x2+x3+x4)) + sin(k*(x1+x2+x3+x4)), k_n=(n+50)/2pi, [0,1]^4"
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libmcbatch_ref.so")


def parse(argv=None):
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
    p.add_argument("--no-configs", action="store_true",
                   help="skip the other-config block (C1/C3/C4/C5 at N=1, C5 weak/strong at N>1)")
    p.add_argument("--c5-fns", type=int, default=10_000, help="configs[4] integrands (strong scaling set)")
    p.add_argument("--c5-samples", type=int, default=10_000_000)
    p.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                   help="weak: every rank integrates its own --n-fns set (default, the driver's scaling run); "
                        "strong: the ranks split one --n-fns set")
    return p.parse_args(argv)


def bench_config(args, world: int) -> dict:
    """The workload identity; both arms print exactly this dict."""
    job = args.n_fns * world if args.scaling == "weak" else args.n_fns
    return {"workload": CONFIG_NAME, "integrands": job,
            "integrands_per_gpu": args.n_fns if args.scaling == "weak" else args.n_fns / world,
            "samples_per_integrand": args.samples, "trials": TRIALS, "seed": SEED, "family": FAMILY,
            "parallelism": f"{args.scaling} dp{world} (integrand shards, no collective)",
            "l2": "GPU arm: 256 MB L2 flush between timed iterations; inputs are ~230 KB of descriptors"}


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
        self.host_group = None
        if world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group(backend=backend)
            self.pg = dist
            # a CPU-side group for waits that must not occupy the GPUs (the
            # NCCL barrier spins a kernel on every rank's device)
            self.host_group = dist.new_group(backend="gloo") if backend != "gloo" else None

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def host_barrier(self):
        if self.pg:
            self.pg.barrier(group=self.host_group)

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

def cpu_info() -> dict:
    """Host CPU model and core counts (the reference arm's hardware)."""
    model, phys = None, set()
    try:
        with open("/proc/cpuinfo") as fh:
            pid = cid = None
            for line in fh:
                k, _, v = line.partition(":")
                k, v = k.strip(), v.strip()
                if k == "model name" and model is None:
                    model = v
                elif k == "physical id":
                    pid = v
                elif k == "core id":
                    cid = v
                elif not k and pid is not None:
                    phys.add((pid, cid))
                    pid = cid = None
            if pid is not None:
                phys.add((pid, cid))
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count()
    return {"model": model, "physical_cores": len(phys) or None, "logical_cpus": os.cpu_count(),
            "usable_cpus": usable}


_ref_lib = None


def load_reference():
    """oracle/_ref/libmcbatch_ref.so — the reference's own sources compiled by
    oracle/Makefile, reached through ref_shim.cpp's ref_run_harmonic (None if
    absent).  Loaded with ctypes only: nothing of the product is imported."""
    global _ref_lib
    if _ref_lib is None and os.path.exists(REF_SO):
        lib = ctypes.CDLL(REF_SO)
        u32, u64, dbl = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double
        lib.ref_run_harmonic.restype = ctypes.c_int
        lib.ref_run_harmonic.argtypes = [u32, u64, u32, u32, u32, u32, ctypes.POINTER(dbl),
                                         ctypes.POINTER(u32), ctypes.POINTER(u32)]
        lib.ref_last_error.restype = ctypes.c_char_p
        _ref_lib = lib
    return _ref_lib


def strided_sample(count: int, step: int, n_total: int = N_FNS):
    """`count` integrands spread over the whole set: stride n_total // count,
    offset rotating with the step so that successive steps cover different k."""
    count = max(1, min(n_total, count))
    stride = max(1, n_total // count)
    return step % stride, count, stride


def cpu_reference_run(count: int, samples: int, step: int = 0):
    """One bounded sample of the workload on the host: the reference's own
    run_batch (workers = 0, every hardware thread) over `count` integrands of
    make_harmonic_job(1000, samples) taken with a stride across the set.
    Returns (samples/s, seconds, kind, threads, sample description)."""
    first, count, stride = strided_sample(count, step)
    lib = load_reference()
    if lib is not None:
        secs, workers, n_ok = ctypes.c_double(), ctypes.c_uint32(), ctypes.c_uint32()
        n = lib.ref_run_harmonic(N_FNS, samples, first, count, stride, 0, ctypes.byref(secs),
                                 ctypes.byref(workers), ctypes.byref(n_ok))
        if n < 0:
            raise RuntimeError("reference run_batch: " + lib.ref_last_error().decode())
        if n_ok.value != n:
            raise RuntimeError(f"reference run_batch: {n - n_ok.value} of {n} integrands failed")
        secs, kind, threads = secs.value, "reference", workers.value
    else:  # the oracle port (test infrastructure) when the reference library is absent
        from paper_2104_10073_b200 import workloads
        from tests import _oracle
        fns, seed, trials = workloads.c2(samples=samples)
        fns = fns[first::stride][:count]
        threads = os.cpu_count() or 1
        t0 = time.perf_counter()
        _oracle.run_direct(fns, seed, trials, n_threads=threads)
        secs = time.perf_counter() - t0
        n, kind = len(fns), "port"
    total = n * samples * TRIALS
    desc = f"integrands n = {first + 1}, {first + 1 + stride}, ... ({n} of {N_FNS}, stride {stride})"
    return total / secs, secs, kind, threads, desc, n


def per_integrand_seconds(samples: int) -> float:
    """Calibration: reference seconds per integrand (a 4-integrand strided sample)."""
    rate, _, _, _, _, _ = cpu_reference_run(4, samples, 0)
    return samples * TRIALS / rate


def cpu_baseline_leg(args) -> dict:
    per_fn = per_integrand_seconds(args.samples)
    n = int(max(1, min(N_FNS, round(args.cpu_seconds / per_fn))))
    rate, secs, kind, threads, desc, _ = cpu_reference_run(n, args.samples, 0)
    return {"value": rate, "unit": "samples/s", "cores": threads, "kind": kind,
            "sample": f"{desc} x {args.samples} samples x {TRIALS} trials ({secs:.1f} s)",
            "cpu": cpu_info()}


def run_reference_arm(args, world, rank):
    if rank != 0:
        return None
    # whole arm within a few minutes: per-step CPU budget, sized by a calibration run
    per_step = max(2.0, min(args.cpu_seconds, 100.0 / (args.steps + 0.25 * args.warmup)))
    per_fn = per_integrand_seconds(args.samples)
    n = int(max(1, min(N_FNS, round(per_step / per_fn))))
    for w in range(args.warmup):
        cpu_reference_run(max(1, n // 4), args.samples, w)
    secs_all, samples_all, descs = [], 0, []
    kind, threads = "port", os.cpu_count()
    for s in range(args.steps):
        rate, secs, kind, threads, desc, m = cpu_reference_run(n, args.samples, s)
        secs_all.append(secs)
        samples_all += m * args.samples * TRIALS
        descs.append(desc)
    value = samples_all / sum(secs_all)
    sample = (f"per step: {descs[0]} x {args.samples} samples x {TRIALS} trials, offset rotating "
              f"with the step ({len(set(descs))} distinct samples over {args.steps} steps); "
              "BatchResult.total_seconds of the reference's run_batch")
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(secs_all) / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args, world),
        "seconds_per_1000_fn_set": N_FNS * args.samples * TRIALS / value,
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads, "kind": kind,
                         "sample": sample, "cpu": cpu_info()},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# ------------------------------------------------------------------ roofline

# Executed mix of the bench kernel's hot loop, k_direct<HARMONIC, 4, 11>, per
# 4-D sample (one loop iteration = one pair of samples; cuobjdump -sass of
# csrc/_obj/direct_harmonic.o through tools/sass_loop.py, committed in
# profiles/r02_k_direct_sass_mix.txt and checked by tests/test_bench_roofline.py):
K_DIRECT_WIDE_PER_SAMPLE = 34   # IMAD.WIDE.U32 (17 per Philox4x32-10 block, 2 blocks)
K_DIRECT_FP64_PER_SAMPLE = 18   # DFMA + DMUL + DADD
# Hardware issue rates per SM sub-partition (SMSP, 4 per SM): IMAD.WIDE runs on
# the FMA-heavy pipe at 32 lanes/clk/SM (a warp instruction every 4 clocks per
# SMSP), FP64 at 64 lanes/clk/SM (every 2 clocks).  The two do not overlap:
# tools/micro/pipe_micro.cu under ncu (profiles/r02_pipe_micro.txt) shows
# fmaheavy-active + fp64-active <= 100 % for any IMAD.WIDE:DFMA mix, while
# IMAD (lo) and DFMA do overlap.  So the ceiling is the SUM of the two costs.
CLK_PER_WIDE_WARP = 4.0
CLK_PER_FP64_WARP = 2.0
N_SM = 148


def alu_roofline(samples_per_s: float, sm_mhz, wide=K_DIRECT_WIDE_PER_SAMPLE, fp64=K_DIRECT_FP64_PER_SAMPLE,
                 clk_per_warp_sample=None):
    """Samples/s against the shared FMA-heavy + FP64 ceiling at the sampled SM clock."""
    if not sm_mhz:
        return None
    if clk_per_warp_sample is None:
        clk_per_warp_sample = wide * CLK_PER_WIDE_WARP + fp64 * CLK_PER_FP64_WARP
    peak = N_SM * 4 * 32 * sm_mhz * 1e6 / clk_per_warp_sample
    return {"achieved": samples_per_s / 1e9, "peak": peak / 1e9, "unit": "G samples/s",
            "frac": samples_per_s / peak, "clk_per_warp_sample": clk_per_warp_sample}


# Hot-loop mix of every k_direct instantiation the other configs launch, per
# loop iteration = one PAIR of samples: (IMAD.WIDE.U32, FP64 ops), keyed by the
# kernel's template arguments (family, dim, variant) as the launch list names
# them (profiles/r02_k_direct_costs.txt; checked against the object files by
# tests/test_bench_roofline.py).  Variants: 0 FAST, 1 FAST unit domain,
# 11 harmonic unit domain + unit coefficients + folded shift.
K_DIRECT_PAIR_MIX = {
    (0, 2, 11): (34, 32), (0, 3, 11): (51, 34), (0, 4, 11): (68, 36), (0, 5, 11): (85, 38),
    (0, 6, 11): (102, 40), (0, 7, 11): (119, 42),
    (2, 2, 0): (34, 18), (3, 3, 0): (51, 24), (2, 2, 1): (34, 10), (3, 3, 1): (51, 12),
}


def mix_clk_per_warp_sample(fns, variant_of) -> float:
    """Sample-weighted FMA-heavy + FP64 clocks per warp-sample of a job whose
    integrand i runs on k_direct<family, dim, variant_of(f)>."""
    clk = samples = 0.0
    for f in fns:
        wide, fp64 = K_DIRECT_PAIR_MIX[(int(f.family), int(f.dim), variant_of(f))]
        clk += f.n_samples * (wide * CLK_PER_WIDE_WARP + fp64 * CLK_PER_FP64_WARP) / 2
        samples += f.n_samples
    return clk / samples


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
    peak = FUSED_BLOCKS_PER_CLK_SM * N_SM * mhz * 1e6
    return {"bound": "alu: Philox + 14-op harmonic, shared IMAD.WIDE/FP64 pipe", "achieved": achieved_blocks_s / 1e9,
            "peak": peak / 1e9, "unit": "G Philox blocks/s", "frac": achieved_blocks_s / peak,
            "peak_source": "tools/micro/split_micro.cu (1.306 blocks/clk/SM) x 148 SMs x sampled SM clock"}


NCU_SUMMARY = "profiles/r02_bench_k_direct_ncu_summary.txt"
NCU_PIPES = "profiles/r02_k_direct_pipes.txt"


def hbm_roofline(traffic_bytes, launch_s):
    """The HBM roofline of the same launch, for reference: measured DRAM bytes
    over the launch time against MEASURED_PEAKS.json's copy bandwidth (the
    schema's "hbm" bound; ~1e-6 here — the kernel is compute-bound)."""
    if traffic_bytes is None or launch_s <= 0:
        return None
    peak = None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
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
    path = os.path.join(ROOT, NCU_SUMMARY)
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


def ncu_pipes():
    """Pipe utilisation of the bench's k_direct launch from the committed ncu
    capture (`key value` lines; None if absent)."""
    out = {}
    try:
        with open(os.path.join(ROOT, NCU_PIPES)) as fh:
            for line in fh:
                parts = line.split()
                if len(parts) == 2 and not line.startswith("#"):
                    try:
                        out[parts[0]] = float(parts[1])
                    except ValueError:
                        pass
    except OSError:
        return None
    return out or None


# ------------------------------------------------------------------ GPU arm

def time_plan(mcb, torch, fns, seed, trials, dev, reps=1, warm=True):
    """Device time of one plan run (CUDA events on the launching stream, L2
    flushed before each timed launch); returns (seconds, info, results)."""
    stream = torch.cuda.current_stream()
    plan = mcb.Plan(fns, seed, trials, device=dev)
    info = plan.info()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{dev}")
    if warm:
        plan.launch(stream.cuda_stream)
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        plan.launch(stream.cuda_stream)
        b.record(stream)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) * 1e-3)
    res = plan.download(stream.cuda_stream)
    plan.close()
    del flush
    return min(times), info, res


def other_configs(mcb, torch, dev, args, peak_blocks, sm_mhz):
    """BASELINE.json configs[0], [2], [3], [4] on this GPU (device-timed plans):
    samples/s, and Philox blocks/s against the live Philox-only ceiling."""
    from paper_2104_10073_b200 import workloads as w
    builders = [
        ("C1", "configs[0]: 100 harmonic 4-D x 1e6 x 10", lambda: w.c1(), 3, True),
        ("C3", "configs[2]: 49 |x1+x2| 2-D + 51 |x1+x2-x3| 3-D, varied domains, 1e6 x 10", lambda: w.c3(), 3, True),
        ("C4", "configs[3]: 4096 harmonic 7-D k_i = 0.01 (i+1) x 1e7 x 10", lambda: w.c4(), 1, False),
        ("C5", f"configs[4] on one GPU: {args.c5_fns} mixed 2-7-D x {args.c5_samples:.0e} x 10",
         lambda: w.c5(samples=args.c5_samples, n_fns=args.c5_fns), 1, False),
    ]
    # kernels of C4/C5 are loaded by a tiny plan first (lazy module loading), so
    # the one timed launch of the big plans needs no warm-up launch of its own
    small, seed, trials = w.c5(samples=70_000, n_fns=16)
    time_plan(mcb, torch, small + w.c4(samples=70_000, n_values=2)[0], seed, trials, dev, reps=1)
    out = {}
    for key, name, build, reps, warm in builders:
        fns, seed, trials = build()
        secs, info, res = time_plan(mcb, torch, fns, seed, trials, dev, reps=reps, warm=warm)
        ok = int((res["status"] == mcb.TRIAL_OK).sum())
        out[key] = {"workload": name, "samples": int(info.total_samples), "seconds": secs,
                    "samples_per_s": info.total_samples / secs,
                    "philox_blocks_per_s": info.philox_blocks / secs,
                    "frac_of_philox_peak": info.philox_blocks / secs / peak_blocks,
                    "ok_trials": ok, "trials_total": len(fns) * trials,
                    "timed_launches": reps, "launches_per_run": int(info.launches_per_run)}
        # the shared FMA-heavy + FP64 ceiling of the job's own kernel mix (C1: the
        # bench kernel; C3: FAST abs on boxes; C4/C5: unit-domain harmonic / abs)
        variant_of = {"C1": lambda f: 11, "C3": lambda f: 0, "C4": lambda f: 11,
                      "C5": lambda f: 11 if int(f.family) == 0 else 1}[key]
        out[key]["alu_roofline"] = alu_roofline(info.total_samples / secs, sm_mhz,
                                                clk_per_warp_sample=mix_clk_per_warp_sample(fns, variant_of))
    return out


def scaling_c5(mcb, torch, dist, dev, args):
    """configs[4] at N > 1 (C5: mixed 2-7-D x 1e7 x 10): weak (c5_fns / 8 per
    rank, global indices) and strong (the c5_fns set split over the ranks),
    one device-timed launch each, max over ranks."""
    from paper_2104_10073_b200 import workloads as w
    out = {}
    per_rank = args.c5_fns // 8
    small, seed, trials = w.c5(samples=70_000, n_fns=16)
    time_plan(mcb, torch, small, seed, trials, dev, reps=1)
    for mode in ("weak", "strong"):
        if mode == "weak":
            every, seed, trials = w.c5(samples=args.c5_samples, n_fns=per_rank * dist.world)
            fns = every[dist.rank * per_rank:(dist.rank + 1) * per_rank]
            job = per_rank * dist.world
        else:
            every, seed, trials = w.c5(samples=args.c5_samples, n_fns=args.c5_fns)
            lo, hi = strong_slice(args.c5_fns, dist.rank, dist.world)
            fns = every[lo:hi]
            job = args.c5_fns
        dist.barrier()
        secs, info, _ = time_plan(mcb, torch, fns, seed, trials, dev, reps=1, warm=False)
        secs = dist.max(secs, device=f"cuda:{dev}")
        samples = job * args.c5_samples * trials
        out[mode] = {"integrands": job, "samples": samples, "seconds": secs, "samples_per_s": samples / secs}
    return out


def run_mcb_arm(args, dist, local):
    import numpy as np
    import torch

    import paper_2104_10073_b200 as mcb
    from paper_2104_10073_b200 import workloads

    # MCB_BENCH_SHARE_GPU=1 (test hook, gloo): ranks share the visible GPUs so the N > 1 code
    # path can run on a one-GPU box; the ranks then compete for one GPU and the numbers mean nothing
    share = os.environ.get("MCB_BENCH_SHARE_GPU") == "1"
    dev = local % torch.cuda.device_count() if share else local
    torch.cuda.set_device(dev)
    if args.scaling == "strong":  # one C2 set, rank r integrates its contiguous slice
        job_fns, seed, trials = workloads.c2(samples=args.samples, n_count=args.n_fns)
        lo, hi = strong_slice(args.n_fns, dist.rank, dist.world)
        fns = job_fns[lo:hi]
    else:
        job_fns, seed, trials = workloads.c2(samples=args.samples, n_count=args.n_fns * dist.world)
        first = shard_first_index(dist.rank, args.n_fns)
        fns = job_fns[first:first + args.n_fns]
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
    clocks = clk.summary()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    kernel_s = sum(step_ms) * 1e-3
    kernel_s_max = dist.max(kernel_s, device=f"cuda:{dev}")
    res = plan.download(stream.cuda_stream)
    plan.close()
    del flush

    # e2e: the reference-facing C-ABI call mcb_run_direct with HOST buffers
    # (descriptor H2D, kernels, result D2H inside the timed region), one call
    # per step over the WHOLE job.  At N > 1 rank 0 makes the call with every
    # GPU in the device list (the product's multi-GPU scheduler: one host
    # thread per device) while the other ranks wait on a CPU-side barrier.
    job_arr = mcb.as_array(job_fns)
    devices = [local % torch.cuda.device_count() if share else r for r in range(dist.world)]
    e2e_times = []
    out = None
    for i in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        dist.host_barrier()
        if dist.rank == 0:
            t0 = time.perf_counter()
            out = mcb.run_direct(job_arr, seed, trials, devices=devices)
            t1 = time.perf_counter()
            if i >= args.warmup:
                e2e_times.append(t1 - t0)
        dist.host_barrier()
    if dist.rank == 0:
        if args.scaling == "strong":
            lo, hi = strong_slice(args.n_fns, 0, dist.world)
        else:
            lo, hi = 0, args.n_fns
        assert out[lo:hi].tobytes() == res.tobytes(), "plan and C-ABI results differ"
    e2e_s = sum(e2e_times)

    job_samples = args.samples * trials * len(job_fns)
    total_samples = job_samples * args.steps
    value = total_samples / kernel_s_max
    e2e_value = total_samples / e2e_s if e2e_s else None

    # roofline of the dominant kernel (k_direct; k_combine is ~8 us of ~55 ms):
    # samples/s of this rank's launches against the hardware-rate ceiling of the
    # kernel's executed mix (IMAD.WIDE + FP64 on pipes that do not overlap)
    rank_rate = info.total_samples / (kernel_s / args.steps)
    # clocks not sampled (--no-clocks): B200's max SM clock
    sm_mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
    alu = alu_roofline(rank_rate, sm_mhz)
    blocks_per_launch = info.philox_blocks
    achieved_blocks = blocks_per_launch / (kernel_s / args.steps)
    peak_blocks = mcb.probe_philox_peak(dev, 50.0)
    traffic = ncu_traffic()
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": dist.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * kernel_s_max / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": bench_config(args, dist.world),
        "seconds_per_1000_fn_set": kernel_s_max / args.steps * 1000 / len(job_fns),
        "run": {"tiles_per_step_per_gpu": int(info.n_tiles), "wall_s_timed_region": wall},
        "e2e": {"value": e2e_value, "unit": "samples/s",
                "h2d_bytes_per_step": ctypes.sizeof(mcb.Integrand) * len(job_fns),
                "d2h_bytes_per_step": int(out.nbytes) if out is not None else int(res.nbytes) * dist.world,
                "path": f"mcb_run_direct(devices={devices}) from rank 0 (C-ABI, host buffers; plan build + "
                        "H2D + kernels + D2H of the whole job)",
                "seconds_per_1000_fn_set": e2e_s / args.steps * 1000 / len(job_fns) if e2e_s else None},
        "gpu_launches": int(info.launches_per_run) * args.steps,
        "roofline": {"bound": "alu: IMAD.WIDE (FMA-heavy pipe) + FP64 pipe, serialised",
                     "achieved": alu["achieved"], "peak": alu["peak"], "unit": alu["unit"],
                     "frac": alu["frac"], "traffic": traffic, "traffic_unit": "DRAM bytes per launch",
                     "per_sample": {"imad_wide": K_DIRECT_WIDE_PER_SAMPLE, "fp64": K_DIRECT_FP64_PER_SAMPLE,
                                    "clk_per_warp_sample_per_smsp": alu["clk_per_warp_sample"]},
                     "note": "achieved = 4-D samples per k_direct<HARMONIC,4> launch / its average duration "
                             "(CUDA events on the launching stream); peak = 148 SMs x 4 SMSPs x 32 lanes x "
                             "sampled SM clock / (34 IMAD.WIDE x 4 clk + 18 FP64 x 2 clk per warp-sample): "
                             "the hardware issue rates of the two pipes, which do not overlap "
                             "(profiles/r02_pipe_micro.txt); instruction counts from the SASS of the hot loop "
                             "(profiles/r02_k_direct_sass_mix.txt); traffic = dram__bytes_read+write of this "
                             "launch from " + NCU_SUMMARY,
                     "sm_mhz": sm_mhz,
                     "ncu_pipes": ncu_pipes(),
                     "philox_only": {"achieved": achieved_blocks / 1e9, "peak": peak_blocks / 1e9,
                                     "unit": "G Philox blocks/s", "frac": achieved_blocks / peak_blocks,
                                     "peak_source": "mcb_probe_philox_peak (Philox-only, same code, live)"},
                     "hbm": hbm_roofline(traffic, kernel_s / args.steps),
                     "fused": fused_roofline(achieved_blocks, clocks)},
        "clocks": clocks,
    }
    if not args.no_configs:
        if dist.world == 1:
            line["configs"] = other_configs(mcb, torch, dev, args, peak_blocks, sm_mhz)
        else:
            line["scaling_c5"] = scaling_c5(mcb, torch, dist, dev, args)
    return line


def main(argv=None):
    args = parse(argv)
    world, rank, local = dist_env()
    if args.impl == "reference":
        line = run_reference_arm(args, world, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    import torch
    backend = "nccl" if torch.cuda.is_available() and os.environ.get("MCB_BENCH_SHARE_GPU") != "1" else "gloo"
    dist = Dist(world, rank, backend)
    line = run_mcb_arm(args, dist, local)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_leg(args)
    dist.close()
    if rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
