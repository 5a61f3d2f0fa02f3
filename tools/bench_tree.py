#!/usr/bin/env python
"""Throughput of the tree method end to end through
mcb_run_direct: host refinement rounds + per-round batched cell launches.
Reports the reference's n_samples (spc per final leaf) per second — the trees
stop below their budget when no leaf stands out — and the samples the kernels
actually draw (split parents included), and the reference's own CPU run_batch on a
bounded sample of the same trees (oracle/_ref, all host threads) when present.

  python tools/bench_tree.py [--fns 200] [--trials 10] [--budget 1000000] [--ref-fns 40]
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
    ap.add_argument("--fns", type=int, default=200)
    ap.add_argument("--trials", type=int, default=10)
    ap.add_argument("--budget", type=int, default=1_000_000)
    ap.add_argument("--spc", type=int, default=2048)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--ref-fns", type=int, default=40)
    ap.add_argument("--integrand", choices=["harmonic", "peak"], default="harmonic",
                    help="harmonic: Fig.1 family (4-D); peak: the C5 gaussian peak DSL program (2-D)")
    args = ap.parse_args()
    import numpy as np

    import paper_2104_10073_b200 as mcb
    from paper_2104_10073_b200 import workloads as w
    mcb.program_jit(2)  # DSL programs: specialised kernels from the first round on

    keep, sources = None, None
    if args.integrand == "peak":
        keep = mcb.Program("exp(-100*((x1-c)^2+(x2-c)^2))", 2, ["c"])
        cs = [0.3 + 0.4 * i / max(1, args.fns - 1) for i in range(args.fns)]
        fns = [mcb.tree(keep.integrand({"c": c}, n_samples=args.budget, index=i), samples_per_cell=args.spc)
               for i, c in enumerate(cs)]
        sources = [f"exp(-100*((x1-{c!r})^2+(x2-{c!r})^2))" for c in cs]
    else:
        fns = [mcb.tree(mcb.harmonic(w.harmonic_k(n), 4, unit_coeffs=True, n_samples=args.budget, index=i),
                        samples_per_cell=args.spc)
               for i, n in enumerate(list(range(1, 101)) * ((args.fns + 99) // 100))][:args.fns]
    for i, f in enumerate(fns):
        f.integrand_index = i
    seed = 20200814
    mcb.run_direct(fns[:2], seed, 2)  # warm-up (module load, buffers)
    times = []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        out = mcb.run_direct(fns, seed, args.trials)
        times.append(time.perf_counter() - t0)
    t = min(times)
    drawn = int(out["n_samples"].sum())
    # n_samples is the reference's count (spc per final leaf); a split re-samples
    # both halves, so the kernels draw (n_leaves - n0) * spc more per tree.  n0
    # (first-pass cells) from one tree's leaves: each first-pass cell is a full
    # binary tree, so sum(2^-depth) over its leaves is 1 (same config for all).
    _, leaves = mcb.tree_refine(fns[0], seed, 0, leaves=True)
    n0 = round(sum(2.0 ** -l.depth for l in leaves))
    actual = drawn + int((out["n_cells"].astype(np.int64) - n0).sum()) * args.spc
    res = {"workload": f"{args.fns} {args.integrand} trees x {args.trials} trials, budget {args.budget}, "
                       f"spc {args.spc}",
           "seconds": t, "samples_drawn": drawn, "samples_per_s": drawn / t,
           "first_pass_cells": n0, "samples_drawn_incl_split_parents": actual,
           "kernel_samples_per_s": actual / t,
           "leaves_mean": float(out["n_cells"].mean()), "max_depth": int(out["max_depth"].max()),
           "budget_exhausted": int(out["budget_exhausted"].sum()),
           "ok": int((out["status"] == mcb.TRIAL_OK).sum())}
    from tests import _oracle
    if args.ref_fns and _oracle.load_ref() is not None:
        sub = fns[:args.ref_fns]
        o, _, _, _, secs = _oracle.ref_run_batch(sub, seed, args.trials, workers=0,
                                                 sources=sources[:args.ref_fns] if sources else None)
        rdrawn = int(o["n_samples"].sum())
        res["reference_cpu"] = {"fns": len(sub), "threads": os.cpu_count(), "seconds": secs,
                                "samples_per_s": rdrawn / secs}
        mine = mcb.run_direct(sub, seed, args.trials)
        res["reference_match_n_samples"] = bool(np.array_equal(mine["n_samples"], o["n_samples"]))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
