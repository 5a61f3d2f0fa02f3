"""Adaptive tree method (ref src/estimator.cpp:184-318,
src/batch.cpp:276-289): initial k^d grid (auto k kept cheap against the
budget), rounds of longest-edge splits of the leaves whose std_error exceeds
mean + sigma * sd, budget exhaustion flagged, combine_cells over the leaves.

CPU: the oracle's tree_refine against the reference's golden run_batch
values (bit-exact) and, in the build container, against the reference
itself leaf by leaf; validation wording.
GPU: the GPU driver (host rounds, cells on the fused kernels) against the
reference's golden trees — leaf rectangles and depths bit-exact, estimates
to 1e-12 — and against the oracle on random family trees; mixed-method
batches; device-list invariance; the reference's tree tests
(tests/test_estimator.cpp:140-192) and acceptance criterion 5
(tests/acceptance.cpp:162-192)."""
import ctypes
import json
import math
import os

import numpy as np
import pytest

from tests import _oracle
from tests.test_oracle import desc_from

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.json")
GAUSS_PEAK_TRUTH = 0.03141592653580133  # (pi/100) erf(5)^2, tests/acceptance.cpp:164


def fx(h):
    return float.fromhex(h)


@pytest.fixture(scope="module")
def tg():
    with open(GOLDEN) as fh:
        return json.load(fh)["tree"]


def refine_kwargs(r):
    kw = dict(r)
    if isinstance(kw.get("sigma_multiplier"), str):
        kw["sigma_multiplier"] = fx(kw["sigma_multiplier"])
    return kw


def batch_fns(mcb, tg):
    fns = []
    for c in tg["batch"]["cases"]:
        f = desc_from(c["desc"])
        mcb.tree(f, **refine_kwargs(c["refine"]))
        fns.append(f)
    return fns


def rel_close(got, want, tol=1e-12, scale=0.0):
    return abs(got - want) <= tol * max(abs(want), scale)


def est_close(got, want, se):
    """Estimates agree to rounding: 1e-12 relative, or 1e-9 of the statistical
    error (a cell mean of an oscillating integrand cancels far below |f|)."""
    return abs(got - want) <= 1e-12 * abs(want) + 1e-9 * se


# ---------------------------------------------------------------- CPU


def test_oracle_tree_batch_matches_reference_golden(mcb, oracle, tg):
    fns = batch_fns(mcb, tg)
    trials = tg["batch"]["trials"]
    out = np.zeros((len(fns), trials), dtype=mcb.TRIAL_DTYPE)
    assert oracle.orc_run_direct(mcb.as_array(fns), len(fns), tg["batch"]["seed"], trials, 2,
                                 out.ctypes.data) == 0
    for i, c in enumerate(tg["batch"]["cases"]):
        for t, want in enumerate(c["per_trial"]):
            got = out[i, t]
            assert float(got["value"]) == fx(want["value"]), (i, t)
            assert float(got["std_error"]) == fx(want["std_error"]), (i, t)
            assert int(got["n_samples"]) == want["n_samples"]
            assert int(got["budget_exhausted"]) == want["budget_exhausted"]


def test_oracle_tree_leaves_match_reference_live(mcb, oracle):
    """The restatement against the reference itself, leaf by leaf (build container)."""
    if _oracle.load_ref() is None:
        pytest.skip("reference build (oracle/_ref) not present")
    rng = np.random.default_rng(11)
    for it in range(12):
        d = int(rng.integers(1, 5))
        fam = int(rng.integers(0, 4))
        if fam == mcb.FAMILY_ABS2 and d < 2 or fam == mcb.FAMILY_ABS3 and d < 3:
            fam = mcb.FAMILY_HARMONIC
        lo = rng.uniform(-1, 0.5, d)
        hi = lo + rng.uniform(0.2, 2.0, d)
        f = mcb.make_integrand(fam, d, k=list(rng.uniform(-9, 9, d)), a=float(rng.uniform(-2, 2)),
                               b=float(rng.uniform(-2, 2)), low=lo, high=hi,
                               n_samples=int(rng.integers(2_000, 120_000)), index=int(rng.integers(0, 9)))
        mcb.tree(f, init_cells_per_dim=int(rng.integers(0, 3)), samples_per_cell=int(rng.integers(64, 3000)),
                 max_depth=int(rng.integers(0, 8)), sigma_multiplier=float(rng.uniform(-1, 2)))
        if fam == mcb.FAMILY_HARMONIC:
            params = {"k": f.k[0], "a": f.a, "b": f.b}
        elif fam == mcb.FAMILY_HARMONIC_VEC:
            params = dict({"a": f.a, "b": f.b}, **{f"k{j + 1}": f.k[j] for j in range(d)})
        else:
            params = {"a": f.a}
        seed, trial, cb = int(rng.integers(0, 2**63)), int(rng.integers(0, 5)), int(rng.integers(0, 50))
        so, lo_ = _oracle.tree_refine(f, seed, trial, cb)
        sr, lr = _oracle.ref_tree_refine(mcb.to_dsl(f), f, params, seed, trial, cb)
        assert (so.status, so.value, so.std_error, so.n_samples, so.budget_exhausted) == \
               (sr.status, sr.value, sr.std_error, sr.n_samples, sr.budget_exhausted), it
        assert len(lo_) == len(lr)
        for a, b in zip(lo_, lr):
            assert list(a.low) == list(b.low) and list(a.high) == list(b.high) and a.depth == b.depth
            assert a.estimate.value == b.estimate.value and a.estimate.std_error == b.estimate.std_error


def test_tree_validation(mcb):
    ok = mcb.tree(mcb.harmonic(1.0, 2, n_samples=10_000))
    assert mcb.validate([ok], 2) == []
    big = mcb.tree(mcb.harmonic(1.0, 3, n_samples=10_000), init_cells_per_dim=200)
    assert (0, "cell grid exceeds configured cap") in mcb.validate([big], 2)
    nan = mcb.tree(mcb.harmonic(1.0, 2, n_samples=10_000), sigma_multiplier=float("nan"))
    assert (0, "sigma_multiplier is NaN") in mcb.validate([nan], 2)
    # defaults without MCB_FLAG_REFINE_CONFIG: a zeroed descriptor is a valid tree
    z = mcb.harmonic(1.0, 2, n_samples=10_000)
    z.method = mcb.METHOD_TREE
    assert mcb.validate([z], 1) == []
    bad = mcb.harmonic(1.0, 2, n_samples=10_000)
    bad.method = 3
    assert (0, "unknown method 3") in mcb.validate([bad], 1)


# ---------------------------------------------------------------- GPU


def program_tree(mcb, c):
    prog = mcb.Program(c["source"], c["dim"], list(c["params"]))
    params = {k: fx(v) for k, v in c["params"].items()}
    f = prog.integrand(params, low=[fx(x) for x in c["low"]], high=[fx(x) for x in c["high"]],
                       n_samples=c["budget"], index=c["index"])
    mcb.tree(f, **c["refine"])
    return prog, f


@pytest.mark.gpu
def test_tree_vs_reference_golden(gpu, tg):
    for c in tg["cases"]:
        prog, f = program_tree(gpu, c)
        st, leaves = gpu.tree_refine(f, c["seed"], c["trial"], c["chunk_base"], leaves=True)
        want = c["estimate"]
        assert st.status == want["status"], c["source"]
        if want["status"] != gpu.TRIAL_OK:
            assert leaves == []
            continue
        assert len(leaves) == want["n_leaves"], c["source"]
        assert st.n_samples == want["n_samples"] and st.n_nonfinite == want["n_nonfinite"]
        assert st.budget_exhausted == want["budget_exhausted"] and st.max_depth == want["max_depth"]
        assert st.nonfinite_warning == want["nonfinite_warning"]
        for got, (lo, hi, depth, val, se, nn) in zip(leaves, c["leaves"]):
            assert [got.low[j] for j in range(c["dim"])] == [fx(x) for x in lo]
            assert [got.high[j] for j in range(c["dim"])] == [fx(x) for x in hi]
            assert got.depth == depth and got.estimate.n_nonfinite == nn
            assert est_close(got.estimate.value, fx(val), fx(se)), c["source"]
            assert rel_close(got.estimate.std_error, fx(se), 1e-9), c["source"]
        assert est_close(st.value, fx(want["value"]), fx(want["std_error"]))
        assert rel_close(st.std_error, fx(want["std_error"]), 1e-9)


@pytest.mark.gpu
def test_tree_batch_vs_reference_golden(gpu, tg):
    fns = batch_fns(gpu, tg)
    trials = tg["batch"]["trials"]
    out = gpu.run_direct(fns, tg["batch"]["seed"], trials)
    for i, c in enumerate(tg["batch"]["cases"]):
        for t, want in enumerate(c["per_trial"]):
            got = out[i, t]
            assert int(got["status"]) == gpu.TRIAL_OK
            assert int(got["n_samples"]) == want["n_samples"], (i, t)
            assert int(got["budget_exhausted"]) == want["budget_exhausted"], (i, t)
            assert est_close(float(got["value"]), fx(want["value"]), fx(want["std_error"])), (i, t)
            assert rel_close(float(got["std_error"]), fx(want["std_error"]), 1e-9), (i, t)
        mean, sd, n_ok = gpu.summarize_trials(out[i])
        assert est_close(mean, fx(c["mean"]), fx(c["per_trial"][0]["std_error"]))


@pytest.mark.gpu
def test_tree_vs_oracle_random_families(gpu, oracle):
    rng = np.random.default_rng(5)
    for it in range(24):
        d = int(rng.integers(1, 6))
        fam = int(rng.integers(0, 4))
        if fam == gpu.FAMILY_ABS2 and d < 2 or fam == gpu.FAMILY_ABS3 and d < 3:
            fam = gpu.FAMILY_HARMONIC_VEC
        lo = rng.uniform(-1, 0.5, d)
        hi = lo + rng.uniform(0.2, 2.0, d)
        f = gpu.make_integrand(fam, d, k=list(rng.uniform(-12, 12, d)), a=float(rng.uniform(-2, 2)),
                               b=float(rng.uniform(-2, 2)), low=lo, high=hi,
                               n_samples=int(rng.integers(5_000, 300_000)), index=int(rng.integers(0, 9)),
                               unit_coeffs=False)
        gpu.tree(f, init_cells_per_dim=int(rng.integers(0, 3)), samples_per_cell=int(rng.integers(100, 5000)),
                 max_depth=int(rng.integers(1, 8)), sigma_multiplier=float(rng.uniform(-0.5, 1.5)))
        seed, trial, cb = int(rng.integers(0, 2**63)), int(rng.integers(0, 5)), int(rng.integers(0, 50))
        so, lo_ = _oracle.tree_refine(f, seed, trial, cb)
        sg, lg = gpu.tree_refine(f, seed, trial, cb, leaves=True)
        assert sg.status == so.status
        assert len(lg) == len(lo_), it
        for a, b in zip(lg, lo_):
            assert list(a.low) == list(b.low) and list(a.high) == list(b.high) and a.depth == b.depth
        assert (sg.n_samples, sg.budget_exhausted, sg.max_depth) == (so.n_samples, so.budget_exhausted,
                                                                     so.max_depth)
        assert est_close(sg.value, so.value, so.std_error), it
        assert rel_close(sg.std_error, so.std_error, 1e-9), it


@pytest.mark.gpu
def test_mixed_methods_batch_and_device_invariance(gpu):
    k3 = 53 / (2 * math.pi)
    fns = [gpu.harmonic(k3, 4, unit_coeffs=True, n_samples=300_000, index=0),
           gpu.tree(gpu.harmonic(k3, 4, unit_coeffs=True, n_samples=300_000, index=1)),
           gpu.stratify(gpu.make_integrand(gpu.FAMILY_ABS2, 2, n_samples=100_000, index=2), cells_per_dim=4),
           gpu.tree(gpu.make_integrand(gpu.FAMILY_ABS3, 3, n_samples=150_000, index=3), samples_per_cell=512),
           gpu.make_integrand(gpu.FAMILY_ABS3, 3, n_samples=70_000, index=4)]
    a = gpu.run_direct(fns, 9, 4)
    b = gpu.run_direct(fns, 9, 4, devices=[0, 0])  # two host threads, LPT shards
    assert a.tobytes() == b.tobytes()
    # each integrand alone gives the same bytes as inside the mixed batch
    for i, f in enumerate(fns):
        assert gpu.run_direct([f], 9, 4).tobytes() == a[i:i + 1].tobytes(), i
    # a tree trial equals the standalone tree_refine with key {seed, i, t, 0}
    for t in range(4):
        st = gpu.tree_refine(fns[1], 9, t, 0)
        assert bytes(st) == a[1, t].tobytes()


@pytest.mark.gpu
def test_reference_tree_unit_tests(gpu):
    """tests/test_estimator.cpp:140-192 on the GPU."""
    const = gpu.Program("5", 2)
    f = gpu.tree(const.integrand(n_samples=100_000))
    st, leaves = gpu.tree_refine(f, 1, 0, 0, leaves=True)
    assert abs(st.value - 5.0) <= 5e-12 and st.std_error == 0.0 and not st.budget_exhausted
    assert st.n_samples <= 100_000

    peak = gpu.Program("exp(-100*((x1-0.5)^2+(x2-0.5)^2))", 2)
    st, leaves = gpu.tree_refine(gpu.tree(peak.integrand(n_samples=100_000)), 21, 0, 0, leaves=True)
    assert abs(st.value - GAUSS_PEAK_TRUTH) <= 3.0 * st.std_error
    vol = sum(np.prod([lf.high[j] - lf.low[j] for j in range(2)]) for lf in leaves)
    assert abs(vol - 1.0) <= 1e-12 and st.n_samples <= 100_000

    off = gpu.Program("exp(-100*((x1-0.3)^2+(x2-0.3)^2))", 2)
    st = gpu.tree_refine(gpu.tree(off.integrand(n_samples=1200), init_cells_per_dim=2, samples_per_cell=256), 31)
    assert st.budget_exhausted and math.isfinite(st.value)

    k = 150.0 / (2.0 * math.pi)
    osc = gpu.harmonic(k, 4, unit_coeffs=True, n_samples=200_000)
    tree = gpu.tree_refine(gpu.tree(gpu.harmonic(k, 4, unit_coeffs=True, n_samples=200_000)), 5, 0, 0)
    direct = gpu.direct_mc(osc, 5, 1, 0)
    band = 3.0 * math.sqrt(tree.std_error ** 2 + direct.std_error ** 2)
    assert abs(tree.value - direct.value) <= band


@pytest.mark.gpu
def test_acceptance_criterion_5(gpu):
    """tests/acceptance.cpp:162-192: tree vs direct on the gaussian peak at an
    equal 1e5 budget over 20 seeds: median std_error tree <= direct, 3-sigma
    coverage >= 18/20 for both."""
    peak = gpu.Program("exp(-100*((x1-0.5)^2+(x2-0.5)^2))", 2)
    tree_se, direct_se, tc, dc = [], [], 0, 0
    for seed in range(20):
        t = gpu.tree_refine(gpu.tree(peak.integrand(n_samples=100_000), samples_per_cell=512), seed, 0, 0)
        d = gpu.direct_mc(peak.integrand(n_samples=100_000), seed, 1, 0)
        tree_se.append(t.std_error)
        direct_se.append(d.std_error)
        tc += abs(t.value - GAUSS_PEAK_TRUTH) <= 3.0 * t.std_error
        dc += abs(d.value - GAUSS_PEAK_TRUTH) <= 3.0 * d.std_error
    assert np.median(tree_se) <= np.median(direct_se)
    assert tc >= 18 and dc >= 18


@pytest.mark.gpu
def test_tree_failure_statuses(gpu):
    dead = gpu.Program("sqrt(-1-x1)", 1)
    st = gpu.tree_refine(gpu.tree(dead.integrand(n_samples=10_000), samples_per_cell=100), 9)
    assert st.status == gpu.TRIAL_ALL_NONFINITE
    capped = gpu.tree(gpu.harmonic(1.0, 2, n_samples=10_000), cell_cap=3)
    assert gpu.tree_refine(capped, 16).status == gpu.TRIAL_CELL_BUDGET
    near = gpu.tree(gpu.harmonic(1.0, 2, n_samples=10_000), init_cells_per_dim=2)
    assert gpu.tree_refine(near, 1, 0, 2**32 - 4).status == gpu.TRIAL_OK  # cells use chunks ..2^32-1
    assert gpu.tree_refine(near, 1, 0, 2**32 - 3).status == gpu.TRIAL_CHUNK_RANGE
    # a batch with one failing tree integrand: the others are unaffected
    out = gpu.run_direct([gpu.tree(gpu.harmonic(1.0, 2, n_samples=10_000, index=0)),
                          gpu.tree(gpu.harmonic(1.0, 2, n_samples=10_000, index=1), cell_cap=3)], 4, 2)
    assert list(out["status"][0]) == [gpu.TRIAL_OK] * 2
    assert list(out["status"][1]) == [gpu.TRIAL_CELL_BUDGET] * 2


_CROSS = r"""
import json, math, sys
sys.path.insert(0, {root!r})
import numpy as np
import paper_2104_10073_b200 as mcb
mcb.program_jit(0)
peak = mcb.Program("exp(-100*((x1-c)^2+(x2-c)^2)) + sqrt(x1*x2)", 2, ["c"])
fns = [mcb.tree(peak.integrand({{"c": 0.3 + 0.05 * i}}, n_samples=60_000, index=i), samples_per_cell=400)
       for i in range(6)]
fns += [mcb.tree(mcb.harmonic(20.0 + i, 3, a=0.5, b=1.5, n_samples=150_000, index=6 + i)) for i in range(4)]
fns += [mcb.tree(mcb.make_integrand(mcb.FAMILY_ABS3, 3, a=1.2, n_samples=90_000, index=10), samples_per_cell=300,
                 sigma_multiplier=0.2, max_depth=9)]
out = mcb.run_direct(fns, 2468, 3)
st, leaves = mcb.tree_refine(fns[0], 99, 1, 5, leaves=True)
print(out.tobytes().hex())
print(bytes(st).hex())
print("".join(bytes(l).hex() for l in leaves))
"""


@pytest.mark.gpu
def test_device_rounds_equal_host_driver(gpu, tmp_path):
    """The device-resident rounds (default) and the host driver over batched
    cell launches (MCB_TREE_DEVICE=0) build identical trees: every byte of
    every result and leaf."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "cross.py"
    script.write_text(_CROSS.format(root=root))
    runs = []
    for mode in ("1", "0"):
        env = dict(os.environ, MCB_TREE_DEVICE=mode)
        r = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, env=env, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        runs.append(r.stdout)
    assert runs[0] == runs[1]
