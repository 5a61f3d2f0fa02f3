"""Generate golden vectors from the REFERENCE ITSELF.

Runs in the build container only: it needs oracle/_ref/libmcbatch_ref.so,
which `make -C oracle ref` compiles from the unmodified reference sources
under /root/reference/proj (src/{expr,sampling,estimator,batch,job_io}.cpp).
Every number in golden.json is produced by the reference's own functions:
  sample_uniform   src/sampling.cpp:102-112
  evaluate         src/expr.cpp:520-553 (on the mcb_to_dsl source)
  direct_mc        src/estimator.cpp:75-92
  tree_refine      src/estimator.cpp:212-318
  run_batch        src/batch.cpp:195-333
  make_harmonic_job / harmonic_closed_form   src/job_io.cpp:336-376
Doubles are stored as float.hex() strings so comparisons are bit-exact.

    python tests/golden/make_golden.py      # rewrites tests/golden/golden.json
"""
from __future__ import annotations

import ctypes
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import paper_2104_10073_b200 as mcb  # noqa: E402  (descriptor structs + mcb_to_dsl only)
from paper_2104_10073_b200 import workloads  # noqa: E402
from tests import _oracle  # noqa: E402

H = float.hex


def desc_json(f):
    return {"family": f.family, "dim": f.dim, "integrand_index": f.integrand_index,
            "flags": f.flags, "n_samples": f.n_samples, "a": H(f.a), "b": H(f.b),
            "k": [H(f.k[j]) for j in range(8)], "low": [H(f.low[j]) for j in range(8)],
            "high": [H(f.high[j]) for j in range(8)], "source": mcb.to_dsl(f)}


def stats_json(st):
    return {"value": H(st.value), "std_error": H(st.std_error), "n_samples": int(st.n_samples),
            "n_nonfinite": int(st.n_nonfinite), "status": int(st.status),
            "nonfinite_warning": int(st.nonfinite_warning)}


def ref_points(ref, low, high, seed, integrand, trial, chunk, count):
    d = len(low)
    out = np.zeros(count * d)
    rc = ref.ref_sample_uniform(d, (ctypes.c_double * d)(*low), (ctypes.c_double * d)(*high), seed,
                                integrand, trial, chunk, count, out.ctypes.data)
    assert rc == 0, ref.ref_last_error()
    return out.reshape(count, d)


def main():
    ref = _oracle.load_ref()
    if ref is None:
        sys.exit("oracle/_ref/libmcbatch_ref.so missing: run `make -C oracle ref` first")
    g = {"generator": "tests/golden/make_golden.py (reference compiled from /root/reference/proj)"}

    # 1. points, including odd-d block straddling, chunk/trial > 0, non-unit domains
    pts_cases = []
    rng = np.random.default_rng(7)
    specs = [(20200814, 0, 0, 0, [0.0] * 4, [1.0] * 4, 8),
             (20200814, 99, 9, 15, [0.0] * 4, [1.0] * 4, 3),
             (7, 1, 0, 0, [0.0] * 3, [1.0] * 3, 5),
             (0, 0, 0, 0, [0.0], [1.0], 6),
             (123, 4, 5, 6, [-1.5, 10.0], [2.25, 20.0], 9),
             (99, 3, 2, 1, [5.0], [5.0 + 1e-6], 7)]
    for d in range(1, 9):
        lo = list(rng.uniform(-3, 0, d))
        hi = [x + w for x, w in zip(lo, rng.uniform(0.5, 4, d))]
        specs.append((int(rng.integers(0, 2**63)), int(rng.integers(0, 5000)), int(rng.integers(0, 10)),
                      int(rng.integers(0, 200)), lo, hi, 11))
    for seed, i, t, c, lo, hi, n in specs:
        p = ref_points(ref, lo, hi, seed, i, t, c, n)
        pts_cases.append({"seed": seed, "integrand": i, "trial": t, "chunk": c,
                          "low": [H(x) for x in lo], "high": [H(x) for x in hi],
                          "points": [[H(x) for x in row] for row in p]})
    g["points"] = pts_cases

    # 2. family values on reference points (evaluate on the lowered source)
    fam = [mcb.harmonic(workloads.harmonic_k(1), 4, unit_coeffs=True),
           mcb.harmonic(3.7, 3, a=0.5, b=-2.0, low=[-1, 0, 2], high=[1, 0.5, 3]),
           mcb.make_integrand(mcb.FAMILY_HARMONIC_VEC, 5, k=[1.5, -2.0, 0.25, 7.0, 3.0], a=1.25,
                              b=0.75),
           mcb.make_integrand(mcb.FAMILY_ABS2, 2, a=1.0),
           mcb.make_integrand(mcb.FAMILY_ABS2, 2, a=1.3, low=[-0.4, 0.0], high=[1.0, 1.4]),
           mcb.make_integrand(mcb.FAMILY_ABS3, 3, a=0.8, low=[0, -0.25, 0], high=[1, 1, 1.5]),
           mcb.harmonic(workloads.harmonic_k(100), 7, unit_coeffs=True)]
    ev = []
    for idx, f in enumerate(fam):
        f.integrand_index = idx
        p = ref_points(ref, [f.low[j] for j in range(f.dim)], [f.high[j] for j in range(f.dim)],
                       20200814, idx, 1, 2, 64)
        vals = np.zeros(64)
        rc = ref.ref_eval_points(mcb.to_dsl(f).encode(), ctypes.byref(f), p.ctypes.data, 64,
                                 vals.ctypes.data)
        assert rc == 0, ref.ref_last_error()
        ev.append({"desc": desc_json(f), "seed": 20200814, "trial": 1, "chunk": 2,
                   "values": [H(v) for v in vals]})
    g["evals"] = ev

    # 3. direct_mc estimates (partial last chunk, chunk_base, trial > 0)
    dm = []
    cases = [(mcb.harmonic(workloads.harmonic_k(1), 4, unit_coeffs=True, n_samples=1_000_000), 20200814, 0, 0),
             (mcb.harmonic(workloads.harmonic_k(100), 4, unit_coeffs=True, n_samples=1_000_000, index=99), 20200814, 9, 0),
             (mcb.harmonic(51.0 / (2 * np.pi), 4, unit_coeffs=True, n_samples=1_000_000), 77, 0, 0),
             (mcb.make_integrand(mcb.FAMILY_ABS2, 2, n_samples=1_000_000), 3, 0, 0),
             (mcb.make_integrand(mcb.FAMILY_ABS3, 3, a=1.0, n_samples=150_001, index=4), 11, 3, 5),
             (mcb.harmonic(0.0, 2, a=7.0, b=1.0, low=[0, 0], high=[2, 2], n_samples=1000, index=2), 1, 0, 0),
             (mcb.harmonic(2.5, 6, a=1.5, b=0.5, low=[-0.5] * 6, high=[0.75] * 6, n_samples=200_003, index=17), 5, 2, 3),
             (mcb.make_integrand(mcb.FAMILY_HARMONIC_VEC, 3, k=[4.0, -1.0, 2.5], a=1.0, b=2.0,
                                 n_samples=100_000, index=8), 42, 1, 0)]
    for f, seed, trial, cb in cases:
        st = mcb.TrialStats()
        rc = ref.ref_direct_mc(mcb.to_dsl(f).encode(), ctypes.byref(f), seed, trial, cb, ctypes.byref(st))
        assert rc == 0, ref.ref_last_error()
        dm.append({"desc": desc_json(f), "seed": seed, "trial": trial, "chunk_base": cb,
                   "estimate": stats_json(st)})
    g["direct_mc"] = dm

    # 4. run_batch: C1 and C3 shapes at reduced sample counts
    rb = []
    for name, (fns, seed, trials) in [("c1_1e5", workloads.c1(100_000)),
                                      ("c3_1e5", workloads.c3(100_000)),
                                      ("c2_first40_2e4", (workloads.c2(20_000)[0][:40], 20200814, 10))]:
        out, mean, sd, ok, _ = _oracle.ref_run_batch(fns, seed, trials, workers=0)
        rb.append({"name": name, "seed": seed, "trials": trials,
                   "descs": [desc_json(f) for f in fns],
                   "per_trial": [[stats_json(_as_stats(out[i, t])) for t in range(trials)]
                                 for i in range(len(fns))],
                   "mean": [H(x) for x in mean], "trial_stddev": [H(x) for x in sd],
                   "ok": [int(x) for x in ok]})
    g["run_batch"] = rb

    # 5. reference known answers (tests/test_job_io.cpp:140-171)
    ks = np.zeros(100)
    seed = ctypes.c_uint64()
    trials = ctypes.c_uint32()
    assert ref.ref_harmonic_job(100, 1_000_000, ks.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                ctypes.byref(seed), ctypes.byref(trials)) == 0
    g["harmonic_job"] = {"k": [H(k) for k in ks], "seed": seed.value, "trials": trials.value,
                         "analytic": [H(ref.ref_analytic_harmonic(n)) for n in range(1, 101)]}

    # 6. stratified method: run_batch Stratified branch (src/batch.cpp:255-275)
    strat = []
    sfns = [mcb.stratify(mcb.harmonic(workloads.harmonic_k(3), 4, unit_coeffs=True, n_samples=100_000, index=0)),
            mcb.stratify(mcb.make_integrand(mcb.FAMILY_ABS2, 2, a=1.3, low=[-0.4, 0.0], high=[1.0, 1.4],
                                            n_samples=50_000, index=1), cells_per_dim=3),
            mcb.stratify(mcb.make_integrand(mcb.FAMILY_ABS3, 3, n_samples=30_000, index=2), cells_per_dim=1),
            mcb.stratify(mcb.make_integrand(mcb.FAMILY_HARMONIC_VEC, 3, k=[2.0, -1.0, 0.5], a=1.5, b=0.5,
                                            low=[-1, 0, 0.5], high=[1, 2, 1.5], n_samples=200_003, index=3)),
            mcb.stratify(mcb.harmonic(0.0, 2, a=3.0, b=1.0, low=[0, 0], high=[1, 2], n_samples=5_000, index=4),
                         cells_per_dim=5),
            mcb.stratify(mcb.harmonic(1.7, 2, a=1.0, b=-2.0, n_samples=300_000, index=5), cells_per_dim=2)]
    out, mean, sd, ok, _ = _oracle.ref_run_batch(sfns, 31, 3, workers=0)
    for i, f in enumerate(sfns):
        strat.append({"desc": desc_json(f), "method": int(f.method), "cells_per_dim": int(f.cells_per_dim),
                      "per_trial": [stats_json(_as_stats(out[i, t])) for t in range(3)],
                      "mean": H(float(mean[i])), "trial_stddev": H(float(sd[i])), "ok": int(ok[i])})
    g["stratified"] = {"seed": 31, "trials": 3, "cases": strat}

    # 7. arbitrary DSL programs (the GPU interpreter's parity anchors)
    g["programs"] = make_program_goldens(ref)

    # 7b. a wider random program sample: dims 1-6, random boxes, 4 parameters
    g["programs_wide"] = make_wide_program_goldens(ref)

    # 8. tree method: tree_refine (src/estimator.cpp:212-318) standalone with
    # leaves, and run_batch's Tree branch (src/batch.cpp:276-289)
    g["tree"] = make_tree_goldens(ref)

    # 9. stratified_mc standalone (src/estimator.cpp:161-182) with leaves
    g["stratified_mc"] = make_stratified_mc_goldens()

    # 10. config scale: C4 / C5 subsets at the configs' own 1e7 samples (153
    # chunks per (integrand, trial)) and near-constant harmonic cases where
    # sum g^2 - (sum g)^2/n would cancel without a good shift
    g["config_scale"] = make_config_scale_goldens(ref)

    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(g, fh, indent=1)
    print("wrote", os.path.join(HERE, "golden.json"))


PROGRAM_CASES = [
    # (source, dim, params, low, high, n_samples, seed, index, trial, chunk_base)
    ("cos(k*(x1+x2+x3+x4)) + sin(k*(x1+x2+x3+x4))", 4, {"k": 8.116902097686662}, [0] * 4, [1] * 4,
     150_000, 20200814, 0, 0, 0),
    ("exp(-50*(x1-0.5)^2)", 1, {}, [0], [1], 100_000, 11, 3, 2, 0),
    ("sqrt(x1)*log(x2+1) + pow(x1, x2)", 2, {}, [0, 0], [1, 2], 70_001, 5, 1, 0, 4),
    ("min(x1,x2) - max(x1, 0.3) + floor(3*x1) / (1 + abs(x2-x1))", 2, {}, [-1, 0], [1, 1.5],
     66_000, 77, 9, 1, 0),
    ("tan(x1) + atan(x2) + asin(x1) - acos(x2)", 2, {}, [0, 0], [0.9, 0.9], 50_000, 3, 2, 0, 0),
    ("log(x1)", 1, {}, [-1], [1], 20_000, 9, 0, 0, 0),
    ("sqrt(-1-x1)", 1, {}, [0], [1], 1_000, 9, 0, 0, 0),
    ("a*x1^2 + b*sin(c*x2) + e - pi*x3", 3, {"a": 1.5, "b": -0.25, "c": 7.0}, [0, -1, 0],
     [2, 1, 0.5], 90_000, 42, 5, 3, 2),
    ("-x1^2 + 2^-x2 - -x3", 3, {}, [-1, -1, -1], [1, 1, 1], 40_000, 8, 0, 0, 0),
    ("7", 2, {}, [0, 0], [2, 2], 1_000, 1, 0, 0, 0),
    ("x1*x2*x3*x4*x5*x6*x7", 7, {}, [0] * 7, [1] * 7, 65_537, 6, 6, 6, 6),
    ("1.5e-3*x1 + 2.E1*x2 + 3.25E+0/x3", 3, {}, [0, 0, 1], [1, 1, 2], 30_000, 2, 0, 1, 0),
]


def random_source(rng, dim, params, depth=0, max_depth=4):
    """Random well-formed DSL source over safe-ish operators."""
    roll = rng.integers(0, 100)
    if depth >= max_depth or roll < 35:
        kind = rng.integers(0, 3)
        if kind == 0:
            return repr(float(np.round(rng.uniform(0, 4), 3)))
        if kind == 1 or not params:
            return f"x{rng.integers(1, dim + 1)}"
        return params[rng.integers(0, len(params))]
    if roll < 45:
        return f"-({random_source(rng, dim, params, depth + 1, max_depth)})"
    if roll < 75:
        op = ["+", "-", "*", "/", "^"][rng.integers(0, 5)]
        l = random_source(rng, dim, params, depth + 1, max_depth)
        r = random_source(rng, dim, params, depth + 1, max_depth)
        return f"({l}){op}({r})"
    if rng.integers(0, 100) < 20:
        fn = ["pow", "min", "max"][rng.integers(0, 3)]
        return f"{fn}({random_source(rng, dim, params, depth + 1, max_depth)}, " \
               f"{random_source(rng, dim, params, depth + 1, max_depth)})"
    fn = ["sin", "cos", "tan", "atan", "exp", "log", "sqrt", "abs", "floor", "asin", "acos"][rng.integers(0, 11)]
    return f"{fn}({random_source(rng, dim, params, depth + 1, max_depth)})"


def make_program_goldens(ref):
    rng = np.random.default_rng(2104)
    cases = list(PROGRAM_CASES)
    for i in range(16):
        src = random_source(rng, 3, ["a", "b"])
        cases.append((src, 3, {"a": float(rng.uniform(-2, 2)), "b": float(rng.uniform(0, 3))},
                      [0, 0, 0], [1, 1, 1], 20_000, 1000 + i, i, i % 3, 0))
    out = []
    for src, dim, params, lo, hi, n, seed, index, trial, cb in cases:
        names = sorted(params)
        cn = (ctypes.c_char_p * max(1, len(names)))(*[x.encode() for x in names])
        vals = (ctypes.c_double * max(1, len(names)))(*[params[x] for x in names])
        lo_c = (ctypes.c_double * dim)(*lo)
        hi_c = (ctypes.c_double * dim)(*hi)
        pts = np.zeros(64 * dim)
        assert ref.ref_sample_uniform(dim, lo_c, hi_c, seed, index, trial, cb, 64, pts.ctypes.data) == 0
        v = np.zeros(64)
        rc = ref.ref_eval_source(src.encode(), dim, cn, vals, len(names), pts.ctypes.data, 64, v.ctypes.data)
        assert rc == 0, (src, ref.ref_last_error())
        st = mcb.TrialStats()
        rc = ref.ref_direct_mc_source(src.encode(), dim, cn, vals, len(names), lo_c, hi_c, n, seed, index,
                                      trial, cb, ctypes.byref(st))
        assert rc == 0, (src, ref.ref_last_error())
        out.append({"source": src, "dim": dim, "params": {k: H(float(x)) for k, x in params.items()},
                    "low": [H(float(x)) for x in lo], "high": [H(float(x)) for x in hi],
                    "n_samples": n, "seed": seed, "index": index, "trial": trial, "chunk_base": cb,
                    "values": [H(float(x)) for x in v], "estimate": stats_json(st)})
    return out


# (source, dim, params, low, high, budget, seed, index, trial, chunk_base, refine kwargs)
TREE_CASES = [
    ("5", 2, {}, [0, 0], [1, 1], 100_000, 1, 0, 0, 0, {}),                       # test_estimator.cpp:140
    ("exp(-100*((x1-0.5)^2+(x2-0.5)^2))", 2, {}, [0, 0], [1, 1], 100_000, 21, 0, 0, 0, {}),  # :153
    ("exp(-100*((x1-0.3)^2+(x2-0.3)^2))", 2, {}, [0, 0], [1, 1], 1_200, 31, 0, 0, 0,
     {"init_cells_per_dim": 2, "samples_per_cell": 256}),                          # :168 budget exhausted
    ("cos(k*(x1+x2+x3+x4)) + sin(k*(x1+x2+x3+x4))", 4, {"k": 150.0 / (2.0 * np.pi)}, [0] * 4, [1] * 4,
     200_000, 5, 0, 0, 0, {}),                                                     # :180
    ("exp(-100*((x1-0.5)^2+(x2-0.5)^2))", 2, {}, [0, 0], [1, 1], 100_000, 0, 0, 0, 0,
     {"samples_per_cell": 512}),                                                   # acceptance.cpp:163
    ("exp(-100*((x1-0.5)^2+(x2-0.5)^2))", 2, {}, [0, 0], [1, 1], 100_000, 7, 0, 0, 0,
     {"samples_per_cell": 512}),
    ("sqrt(x1-0.6) + x2", 2, {}, [0, 0], [1, 1], 50_000, 4, 2, 1, 0, {"samples_per_cell": 512}),  # dead leaves
    ("sqrt(-1-x1)", 1, {}, [0], [1], 10_000, 9, 0, 0, 0, {"samples_per_cell": 100}),  # all dead
    ("a*x1*x2 + sin(b*x3)", 3, {"a": 2.5, "b": 9.0}, [0, -1, 0], [1, 1, 2], 80_000, 12, 3, 2, 7,
     {"sigma_multiplier": -0.5, "samples_per_cell": 300}),                         # eager splitting
    ("x1^3 - x2", 2, {}, [-1, -1], [1, 1], 60_000, 13, 0, 0, 0, {"max_depth": 0}),  # no refinement
    ("abs(x1-x2)", 2, {}, [0, 0], [1, 1], 90_000, 14, 0, 0, 0,
     {"init_cells_per_dim": 3, "max_depth": 2, "samples_per_cell": 1000}),
    ("exp(x1)", 2, {}, [0, 0], [1, 1], 10_000, 15, 0, 0, 0, {"init_cells_per_dim": 4, "cell_cap": 10}),
    ("exp(x1)", 2, {}, [0, 0], [1, 1], 10_000, 16, 0, 0, 0, {"cell_cap": 3}),
    ("1/(x1-0.5)", 1, {}, [0], [1], 40_000, 17, 0, 0, 0, {"samples_per_cell": 70_000}),  # 2-chunk cells
]


def tree_desc(f, kw):
    return mcb.tree(f, **kw)


def make_tree_goldens(ref):
    out = []
    for src, dim, params, lo, hi, budget, seed, index, trial, cb, kw in TREE_CASES:
        prog = mcb.Program(src, dim, list(params))
        f = tree_desc(prog.integrand(params, low=lo, high=hi, n_samples=budget, index=index), kw)
        st, leaves = _oracle.ref_tree_refine(src, f, params, seed, trial, cb)
        out.append({"source": src, "dim": dim, "params": {k: H(float(x)) for k, x in params.items()},
                    "low": [H(float(x)) for x in lo], "high": [H(float(x)) for x in hi],
                    "budget": budget, "seed": seed, "index": index, "trial": trial, "chunk_base": cb,
                    "refine": kw, "estimate": dict(stats_json(st), budget_exhausted=int(st.budget_exhausted),
                                                    n_leaves=len(leaves), max_depth=int(st.max_depth)),
                    "leaves": [[[H(l.low[j]) for j in range(dim)], [H(l.high[j]) for j in range(dim)],
                                int(l.depth), H(l.estimate.value), H(l.estimate.std_error),
                                int(l.estimate.n_nonfinite)] for l in leaves]})
    # run_batch Tree branch on family integrands, 3 trials
    fns = [mcb.tree(mcb.harmonic(150 / (2 * np.pi), 4, unit_coeffs=True, n_samples=100_000, index=0)),
           mcb.tree(mcb.make_integrand(mcb.FAMILY_ABS3, 3, a=2.0, low=[-1, 0, 0.5], high=[1, 2, 3],
                                       n_samples=60_000, index=1), samples_per_cell=512, sigma_multiplier=0.5),
           mcb.tree(mcb.harmonic(3.0, 2, a=0.5, b=-1.5, n_samples=1_200, index=2), init_cells_per_dim=2,
                    samples_per_cell=256),
           mcb.tree(mcb.make_integrand(mcb.FAMILY_HARMONIC_VEC, 3, k=[2.0, -1.0, 9.5], a=1.5, b=0.5,
                                       low=[-1, 0, 0.5], high=[1, 2, 1.5], n_samples=150_000, index=3),
                    samples_per_cell=1024, max_depth=3),
           mcb.tree(mcb.make_integrand(mcb.FAMILY_ABS2, 2, n_samples=30_000, index=4), sigma_multiplier=0.0,
                    samples_per_cell=200)]
    o, mean, sd, ok, _ = _oracle.ref_run_batch(fns, 77, 3, workers=0)
    batch = [{"desc": desc_json(f), "refine": {"init_cells_per_dim": int(f.cells_per_dim),
                                                "samples_per_cell": int(f.samples_per_cell),
                                                "max_depth": int(f.max_depth),
                                                "sigma_multiplier": H(f.sigma_multiplier)},
              "per_trial": [dict(stats_json(_as_stats(o[i, t])), budget_exhausted=int(o[i, t]["budget_exhausted"]))
                            for t in range(3)],
              "mean": H(float(mean[i])), "trial_stddev": H(float(sd[i])), "ok": int(ok[i])}
             for i, f in enumerate(fns)]
    return {"cases": out, "batch": {"seed": 77, "trials": 3, "cases": batch}}


STRAT_MC_CASES = [
    # (source, dim, params, low, high, cells_per_dim, spc, seed, index, trial, chunk_base, cell_cap)
    ("sin(x1)*x2", 2, {}, [0.25, -1.0], [0.75, 3.0], 1, 5000, 11, 2, 0, 0, 0),   # test_estimator.cpp:87-97
    ("exp(-a*((x1-0.5)^2+(x2-0.3)^2)) + x1*x2", 2, {"a": 20.0}, [0, 0], [1, 1], 3, 333, 123, 5, 0, 0, 0),
    ("cos(k*(x1+x2+x3+x4)) + sin(k*(x1+x2+x3+x4))", 4, {"k": 13.0}, [0] * 4, [1] * 4, 3, 700, 9, 1, 2, 5, 0),
    ("5", 3, {}, [0, 0, 0], [2, 1, 1], 4, 100, 1, 0, 0, 0, 0),
    ("log(x1)", 1, {}, [-1], [1], 4, 1000, 9, 0, 0, 0, 0),                        # dead cells
    ("x1", 2, {}, [0, 0], [1, 1], 10, 10, 3, 0, 0, 0, 50),                        # past the cap
    ("abs(x1-x2)*x3", 3, {}, [-1, 0, 0], [1, 1, 2], 2, 70_000, 4, 3, 1, 0, 0),    # 2-chunk cells
]


def make_stratified_mc_goldens():
    out = []
    for src, dim, params, lo, hi, k, spc, seed, index, trial, cb, cap in STRAT_MC_CASES:
        prog = mcb.Program(src, dim, list(params))
        f = prog.integrand(params, low=lo, high=hi, n_samples=max(2, spc), index=index)
        st, leaves = _oracle.ref_stratified_mc(src, f, params, k, spc, seed, trial, cb, cap)
        out.append({"source": src, "dim": dim, "params": {kk: H(float(x)) for kk, x in params.items()},
                    "low": [H(float(x)) for x in lo], "high": [H(float(x)) for x in hi], "cells_per_dim": k,
                    "samples_per_cell": spc, "seed": seed, "index": index, "trial": trial, "chunk_base": cb,
                    "cell_cap": cap, "estimate": dict(stats_json(st), n_leaves=len(leaves)),
                    "leaves": [[[H(l.low[j]) for j in range(dim)], [H(l.high[j]) for j in range(dim)],
                                H(l.estimate.value), H(l.estimate.std_error)] for l in leaves]})
    return out


def make_wide_program_goldens(ref):
    rng = np.random.default_rng(91)
    out = []
    for i in range(64):
        dim = int(rng.integers(1, 7))
        names = ["a", "b", "c", "d"][: int(rng.integers(0, 5))]
        src = random_source(rng, dim, names, max_depth=int(rng.integers(2, 6)))
        params = {n: float(np.round(rng.uniform(-3, 3), 6)) for n in names}
        lo = np.round(rng.uniform(-2, 1, dim), 4)
        hi = lo + np.round(rng.uniform(0.25, 3, dim), 4)
        seed, index, trial, cb = int(rng.integers(0, 2**40)), i, int(rng.integers(0, 5)), int(rng.integers(0, 4))
        n = int(rng.integers(2, 90_000))
        nm = sorted(params)
        cn = (ctypes.c_char_p * max(1, len(nm)))(*[x.encode() for x in nm])
        vals = (ctypes.c_double * max(1, len(nm)))(*[params[x] for x in nm])
        lo_c, hi_c = (ctypes.c_double * dim)(*lo), (ctypes.c_double * dim)(*hi)
        pts = np.zeros(32 * dim)
        assert ref.ref_sample_uniform(dim, lo_c, hi_c, seed, index, trial, cb, 32, pts.ctypes.data) == 0
        v = np.zeros(32)
        assert ref.ref_eval_source(src.encode(), dim, cn, vals, len(nm), pts.ctypes.data, 32, v.ctypes.data) == 0
        st = mcb.TrialStats()
        assert ref.ref_direct_mc_source(src.encode(), dim, cn, vals, len(nm), lo_c, hi_c, n, seed, index, trial, cb,
                                        ctypes.byref(st)) == 0
        out.append({"source": src, "dim": dim, "params": {k: H(x) for k, x in params.items()},
                    "low": [H(float(x)) for x in lo], "high": [H(float(x)) for x in hi], "n_samples": n,
                    "seed": seed, "index": index, "trial": trial, "chunk_base": cb,
                    "values": [H(float(x)) for x in v], "estimate": stats_json(st)})
    return out


# C4 (parameter_scan of the 7-D harmonic, k_i = 0.01 (i+1)): 8 of the 4096
# values, k = 0.01 ... 40.96, with their scan positions as integrand indices.
C4_SUBSET = [0, 4, 19, 99, 511, 1023, 2047, 4095]
# C5 (10^4 integrands cycling abs2/abs3/harmonic d = 2..7): n = 617 i cycles
# all 8 kinds twice (617 = 1 mod 8).
C5_SUBSET = [617 * i for i in range(16)]


def threshold_cases():
    """Near-constant harmonic integrands (argument sweep 0.05-0.1 rad at an
    extremum of a*cos + b*sin): var/mean^2 ~ 1e-7, the regime where an
    unshifted sum of squares loses the std_error."""
    q = math.pi / 4
    return [
        mcb.harmonic(1.0, 1, a=1.0, b=0.0, low=[0.0], high=[0.05], n_samples=2_000_000, index=0),
        mcb.harmonic(1.0, 1, a=1.0, b=0.0, low=[0.0], high=[0.1], n_samples=2_000_000, index=1),
        mcb.harmonic(0.05 / 4, 4, a=1.0, b=0.0, n_samples=2_000_000, index=2),
        mcb.harmonic(0.1 / 4, 4, a=1.0, b=0.0, n_samples=2_000_000, index=3),
        mcb.harmonic(1.0, 2, a=0.0, b=1.0, low=[q - 0.0125] * 2, high=[q + 0.0125] * 2, n_samples=2_000_000,
                     index=4),
        mcb.harmonic(0.1 / 7, 7, a=1.0, b=0.0, n_samples=2_000_000, index=5),
        mcb.harmonic(1.0, 1, a=1.0, b=0.0, low=[-0.025], high=[0.025], n_samples=2_000_000, index=6),
        mcb.make_integrand(mcb.FAMILY_HARMONIC_VEC, 3, k=[0.01, 0.02, 0.005], a=2.0, b=0.0,
                           n_samples=2_000_000, index=7),
        mcb.harmonic(1.0, 4, a=3.0, b=0.5, low=[0.1] * 4, high=[0.1125] * 4, n_samples=2_000_000, index=8),
    ]


def config_scale_specs():
    c4, seed4, _ = workloads.c4(samples=10_000_000)
    c5, seed5, _ = workloads.c5(samples=10_000_000, n_fns=C5_SUBSET[-1] + 1)
    return ([("c4", c4[i], seed4) for i in C4_SUBSET] + [("c5", c5[n], seed5) for n in C5_SUBSET] +
            [("threshold", f, 97) for f in threshold_cases()])


def make_config_scale_goldens(ref):
    from concurrent.futures import ThreadPoolExecutor
    specs = config_scale_specs()
    trials = 2

    def one(job):
        (_, f, seed), t = job
        st = mcb.TrialStats()
        rc = ref.ref_direct_mc(mcb.to_dsl(f).encode(), ctypes.byref(f), seed, t, 0, ctypes.byref(st))
        assert rc == 0, ref.ref_last_error()
        return stats_json(st)

    jobs = [(sp, t) for sp in specs for t in range(trials)]
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:  # ctypes drops the GIL
        res = list(ex.map(one, jobs))
    out = []
    for i, (group, f, seed) in enumerate(specs):
        out.append({"group": group, "desc": desc_json(f), "seed": seed,
                    "per_trial": res[i * trials:(i + 1) * trials]})
    return {"trials": trials, "chunk_base": 0, "cases": out}


def _as_stats(row):
    st = mcb.TrialStats()
    st.value, st.std_error = float(row["value"]), float(row["std_error"])
    st.n_samples, st.n_nonfinite = int(row["n_samples"]), int(row["n_nonfinite"])
    st.status, st.nonfinite_warning = int(row["status"]), int(row["nonfinite_warning"])
    return st


if __name__ == "__main__":
    main()
