#!/usr/bin/env python
"""Measurement of every SURVEY.md §8(f) row built beside the direct path, each
against the reference's own CPU implementation (oracle/_ref, all host
threads) on a bounded sample of the same workload:

  programs    C2 as DSL programs (GPU interpreter) + a 2-D gaussian-peak program set
  stratified  C2 with the stratified method (auto k: 8^4 cells of 244 samples)
  job         `mcb run` on the gen-fig1 job (100 x 1e6 x 10) vs the reference's run_command
  tree        Fig.1 harmonic trees (1e6 budget) and gaussian-peak trees (1e5, spc 512)

GPU numbers: device-resident plans timed with CUDA events (programs,
stratified), or end to end through mcb_run_direct / the CLI (tree, job).
One JSON line per row.

  python tools/bench_rows.py [--rows programs,stratified,job,tree]
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

FIG1 = "cos(k*(x1+x2+x3+x4)) + sin(k*(x1+x2+x3+x4))"


def plan_rate(mcb, fns, seed, trials, reps=3):
    import torch
    stream = torch.cuda.current_stream()
    plan = mcb.Plan(fns, seed, trials)
    info = plan.info()
    plan.launch(stream.cuda_stream)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        plan.launch(stream.cuda_stream)
        b.record(stream)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3)
    res = plan.download(stream.cuda_stream)
    plan.close()
    return {"samples": info.total_samples, "seconds": best, "samples_per_s": info.total_samples / best,
            "ok_trials": int((res["status"] == mcb.TRIAL_OK).sum())}


def ref_rate(fns, seed, trials, sources=None):
    from tests import _oracle
    if _oracle.load_ref() is None:
        return None
    out, _, _, _, secs = _oracle.ref_run_batch(fns, seed, trials, workers=0, sources=sources)
    n = int(out["n_samples"].sum())
    return {"integrands": len(fns), "threads": os.cpu_count(), "samples": n, "seconds": secs,
            "samples_per_s": n / secs}


def row_programs(mcb, w):
    mcb.program_jit(2)  # measure the specialised kernels (compiled before the first launch)
    fns, seed, trials = w.c2()
    prog = mcb.Program(FIG1, 4, ["k"])
    pf = [prog.integrand({"k": f.k[0]}, n_samples=f.n_samples, index=f.integrand_index) for f in fns]
    gpu = plan_rate(mcb, pf, seed, trials)
    ref = ref_rate(pf[:6], seed, trials, sources=[FIG1.replace("k", repr(f.k[0])) for f in pf[:6]])
    peak = mcb.Program("exp(-100*((x1-c)^2+(x2-c)^2)) + sqrt(x1*x2)", 2, ["c"])
    cs = [0.2 + 0.6 * i / 999 for i in range(1000)]
    pk = [peak.integrand({"c": c}, n_samples=1_000_000, index=i) for i, c in enumerate(cs)]
    gpu_peak = plan_rate(mcb, pk, 7, 10)
    ref_peak = ref_rate(pk[:6], 7, 10, sources=[f"exp(-100*((x1-{c!r})^2+(x2-{c!r})^2)) + sqrt(x1*x2)"
                                                   for c in cs[:6]])
    return {"row": "programs (GPU bytecode interpreter)",
            "fig1_as_program": {"workload": "C2 sources, 1000 x 1e6 x 10", "gpu": gpu, "reference_cpu": ref},
            "peak_program": {"workload": "1000 x 2-D gaussian peak + sqrt, 1e6 x 10", "gpu": gpu_peak,
                             "reference_cpu": ref_peak}}


def row_stratified(mcb, w):
    fns, seed, trials = w.c2()
    for f in fns:
        mcb.stratify(f)
    gpu = plan_rate(mcb, fns, seed, trials)
    ref = ref_rate(fns[:6], seed, trials)
    return {"row": "stratified", "workload": "C2, auto k (8^4 cells x 244 samples)", "gpu": gpu,
            "reference_cpu": ref}


def row_job(mcb, w):
    from tests import _oracle
    cli = os.path.join(ROOT, "paper_2104_10073_b200", "mcb")
    d = tempfile.mkdtemp()
    job, out_gpu, out_ref = (os.path.join(d, x) for x in ("fig1.json", "gpu.csv", "ref.csv"))
    subprocess.run([cli, "gen-fig1", "--out", job], check=True)
    subprocess.run([cli, "run", job, "--out", out_gpu], check=True, capture_output=True)  # warm
    t0 = time.perf_counter()
    subprocess.run([cli, "run", job, "--out", out_gpu], check=True, capture_output=True)
    t_gpu = time.perf_counter() - t0
    chk = subprocess.run([cli, "check-fig1", out_gpu], capture_output=True, text=True)
    res = {"row": "job files / CSV / CLI", "workload": "gen-fig1 job: 100 x 1e6 x 10 (1e9 samples)",
           "gpu_cli": {"seconds": t_gpu, "samples_per_s": 1e9 / t_gpu,
                       "check_fig1": chk.stdout.strip().splitlines()[-1]}}
    ref = _oracle.load_ref()
    if ref is not None:
        t0 = time.perf_counter()
        rc = ref.ref_run_command(job.encode(), out_ref.encode(), 0)
        t_ref = time.perf_counter() - t0
        res["reference_run_command"] = {"rc": rc, "threads": os.cpu_count(), "seconds": t_ref,
                                        "samples_per_s": 1e9 / t_ref}
    return res


def row_tree():
    out = {"row": "tree"}
    for name, extra in [("harmonic", ["--fns", "200", "--budget", "1000000"]),
                        ("peak", ["--integrand", "peak", "--fns", "200", "--budget", "100000", "--spc", "512"])]:
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "bench_tree.py"), *extra],
                           capture_output=True, text=True, check=True)
        out[name] = json.loads(r.stdout.strip().splitlines()[-1])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", default="programs,stratified,job,tree")
    args = ap.parse_args()
    import paper_2104_10073_b200 as mcb
    from paper_2104_10073_b200 import workloads as w
    for row in args.rows.split(","):
        if row == "programs":
            r = row_programs(mcb, w)
        elif row == "stratified":
            r = row_stratified(mcb, w)
        elif row == "job":
            r = row_job(mcb, w)
        else:
            r = row_tree()
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
