#!/usr/bin/env python
"""Throughput of every BASELINE.json config on one GPU (device-resident plan,
CUDA events on the launching stream).  Not the driver's bench line (that is
bench.py on configs[1]); this is the per-config table for DESIGN.md.

  python tools/bench_configs.py [--reps 3] [--configs c1,c2,c3,c4,c5] [--c5-fns 10000]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    ap.add_argument("--c5-fns", type=int, default=10000)
    ap.add_argument("--c4-trials", type=int, default=10)
    ap.add_argument("--reference-seconds", type=float, default=0.0,
                    help="also time the reference's own run_batch (oracle/_ref, all host threads) on a "
                         "deterministic prefix of each config sized to about this many seconds")
    args = ap.parse_args()
    import torch

    import paper_2104_10073_b200 as mcb
    from paper_2104_10073_b200 import workloads as w

    def as_program(fns_seed_trials):
        fns, seed, trials = fns_seed_trials
        prog = mcb.Program("cos(k*(x1+x2+x3+x4)) + sin(k*(x1+x2+x3+x4))", 4, ["k"])
        out = [prog.integrand({"k": f.k[0]}, n_samples=f.n_samples, index=f.integrand_index) for f in fns]
        out.append(prog)  # keep alive
        return out, seed, trials

    def stratified(fns_seed_trials):
        fns, seed, trials = fns_seed_trials
        for f in fns:
            if isinstance(f, mcb.Integrand):
                mcb.stratify(f)
        return fns, seed, trials

    builders = {
        "c1_strat": lambda: stratified(w.c1()),
        "c2_strat": lambda: stratified(w.c2()),
        "c3_strat": lambda: stratified(w.c3()),
        "c1_program": lambda: as_program(w.c1()),
        "c2_program_strat": lambda: stratified(as_program(w.c2())),
        "c2_program": lambda: as_program(w.c2()),
        "c1": lambda: w.c1(),
        "c2": lambda: w.c2(),
        "c3": lambda: w.c3(),
        "c4": lambda: w.c4(trials=args.c4_trials),
        "c5": lambda: w.c5(n_fns=args.c5_fns),
    }
    stream = torch.cuda.current_stream()
    # program configs: specialised kernels compiled before the first launch
    # (MCB_PROGRAM_JIT=0 in the environment measures the bytecode interpreter)
    mcb.program_jit(0 if os.environ.get("MCB_PROGRAM_JIT") == "0" else 2)
    peak = mcb.probe_philox_peak(0, 50.0)
    out = {"philox_peak_blocks_per_s": peak}
    for name in args.configs.split(","):
        fns, seed, trials = builders[name]()
        keep = [x for x in fns if isinstance(x, mcb.Program)]
        fns = [x for x in fns if not isinstance(x, mcb.Program)]
        plan = mcb.Plan(fns, seed, trials)
        info = plan.info()
        plan.launch(stream.cuda_stream)  # warm-up (module load)
        torch.cuda.synchronize()
        times = []
        for _ in range(args.reps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            plan.launch(stream.cuda_stream)
            b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b) * 1e-3)
        t = min(times)
        res = plan.download(stream.cuda_stream)
        plan.close()
        ok = int((res["status"] == mcb.TRIAL_OK).sum())
        out[name] = {"integrands": len(fns), "trials": trials, "samples": info.total_samples,
                     "groups": info.n_groups, "tiles": info.n_tiles, "seconds": t,
                     "samples_per_s": info.total_samples / t,
                     "philox_blocks_per_s": info.philox_blocks / t,
                     "frac_of_philox_peak": info.philox_blocks / t / peak,
                     "ok_trials": ok}
        if args.reference_seconds > 0 and not keep:
            out[name]["reference_cpu"] = reference_rate(fns, seed, trials, args.reference_seconds)
            out[name]["speedup_vs_reference"] = out[name]["samples_per_s"] / out[name]["reference_cpu"]["samples_per_s"]
        print(name, json.dumps(out[name]), flush=True)
    print(json.dumps(out))


def reference_rate(fns, seed, trials, target_s):
    """The reference's run_batch on the first integrands of the config: a
    calibration run on one, then a prefix sized to ~target_s."""
    import os

    from tests import _oracle
    if _oracle.load_ref() is None:
        return None
    _, _, _, _, secs = _oracle.ref_run_batch(fns[:1], seed, trials, workers=0)
    n = int(max(1, min(len(fns), target_s / max(secs, 1e-3))))
    out, _, _, _, secs = _oracle.ref_run_batch(fns[:n], seed, trials, workers=0)
    samples = int(out["n_samples"].sum())
    return {"integrands": n, "of": len(fns), "threads": os.cpu_count(), "seconds": secs,
            "samples_per_s": samples / secs}


if __name__ == "__main__":
    main()
