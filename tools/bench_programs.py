#!/usr/bin/env python
"""DSL-program throughput on one GPU, interpreter and specialised (JIT) kernels,
for kernel-variant comparisons (select a library with MCB_LIB=...):

  C2 as programs      cos(k*(x1+x2+x3+x4)) + sin(k*(x1+x2+x3+x4)), 1000 x 1e6 x 10
  peak                exp(-100*((x1-c)^2+(x2-c)^2)) + sqrt(x1*x2), 1000 x 1e6 x 10
  peak on a box       the same on [0.1, 0.9]^2 (non-unit domain)

Device-resident plans timed with CUDA events (best of --reps).  One JSON line.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

FIG1 = "cos(k*(x1+x2+x3+x4)) + sin(k*(x1+x2+x3+x4))"
PEAK = "exp(-100*((x1-c)^2+(x2-c)^2)) + sqrt(x1*x2)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--modes", default="interp,jit")
    args = ap.parse_args()
    import paper_2104_10073_b200 as mcb
    from paper_2104_10073_b200 import workloads as w
    from bench_rows import plan_rate

    fns, seed, trials = w.c2()
    fig1 = mcb.Program(FIG1, 4, ["k"])
    peak = mcb.Program(PEAK, 2, ["c"])
    cs = [0.2 + 0.6 * i / 999 for i in range(1000)]
    sets = {
        "c2_program": ([fig1.integrand({"k": f.k[0]}, n_samples=f.n_samples, index=f.integrand_index)
                        for f in fns], seed),
        "peak": ([peak.integrand({"c": c}, n_samples=1_000_000, index=i) for i, c in enumerate(cs)], 7),
        "peak_box": ([peak.integrand({"c": c}, n_samples=1_000_000, index=i, low=[0.1, 0.1], high=[0.9, 0.9])
                      for i, c in enumerate(cs)], 7),
    }
    out = {"lib": os.environ.get("MCB_LIB", "in-tree")}
    for mode in args.modes.split(","):
        mcb.program_jit(0 if mode == "interp" else 2)
        for name, (integrands, sd) in sets.items():
            r = plan_rate(mcb, integrands, sd, trials, reps=args.reps)
            out[f"{name}/{mode}"] = round(r["samples_per_s"] / 1e9, 2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
