"""GPU parity: the sm_100a path (through the C-ABI) against the oracle and the
reference's golden vectors.

Bars (BASELINE.json north_star):
  * points: BIT-EXACT vs sample_uniform (src/sampling.cpp:102-112);
  * per-(integrand, trial) value: |gpu - ref| <= max(1e-9 |ref|, 1e-12 V RMS(f)),
    the absolute floor (near-zero means) taken from the reference's own
    estimate: (V RMS(f))^2 = value^2 + std_error^2 n;
  * std_error: 1e-9 relative;  n_samples / n_nonfinite: identical;
  * results byte-identical for any device list (GPU-count invariance).
Every comparison records its deviation in units of its tolerance; the
largest per test is printed (pytest -s) — tests/_deviation.py.
"""
import json
import math
import os

import numpy as np
import pytest

from tests import _oracle
from tests._deviation import REL, check_stats, close, record  # noqa: F401

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.json")


def fx(h):
    return float.fromhex(h)


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as fh:
        return json.load(fh)


# ------------------------------------------------------------------ sampler

def test_points_bit_exact_golden(gpu, golden):
    for case in golden["points"]:
        lo = [fx(x) for x in case["low"]]
        hi = [fx(x) for x in case["high"]]
        want = np.array([[fx(x) for x in row] for row in case["points"]])
        got = gpu.debug_points(case["seed"], case["integrand"], case["trial"], case["chunk"], 0,
                               len(want), lo, hi)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), case


def test_points_bit_exact_oracle_sweep(gpu):
    rng = np.random.default_rng(5)
    for d in range(1, 9):
        for _ in range(3):
            lo = rng.uniform(-5, 5, d)
            hi = lo + rng.uniform(1e-6, 10, d)
            seed = int(rng.integers(0, 2**63))
            idx, trial = int(rng.integers(0, 2**32)), int(rng.integers(0, 1000))
            chunk = int(rng.integers(0, 2**32))
            first = int(rng.integers(0, 60000))
            n = 777
            got = gpu.debug_points(seed, idx, trial, chunk, first, n, list(lo), list(hi))
            want = _oracle.sample_uniform(list(lo), list(hi), seed, idx, trial, chunk, first, n)
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (d, seed)


def test_points_unit_and_edge_domains(gpu):
    for lo, hi in [([0.0], [1.0]), ([5.0], [5.0 + 1e-6]), ([-1.5, 10], [2.25, 20]),
                   ([0.0] * 7, [1.0] * 7), ([-1e300], [1e300])]:
        got = gpu.debug_points(20200814, 3, 2, 1, 0, 4096, lo, hi)
        want = _oracle.sample_uniform(lo, hi, 20200814, 3, 2, 1, 0, 4096)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
        assert (got >= np.array(lo)).all() and (got < np.array(hi)).all() or hi[0] == 1e300


# ------------------------------------------------------------------ evaluator

def _families(mcb):
    from paper_2104_10073_b200 import workloads
    return [
        mcb.harmonic(workloads.harmonic_k(1), 4, unit_coeffs=True),                  # FAST unit dom/coef
        mcb.harmonic(workloads.harmonic_k(100), 7, unit_coeffs=True),
        mcb.harmonic(3.7, 3, a=0.5, b=-2.0, low=[-1, 0, 2], high=[1, 0.5, 3]),       # FAST general
        mcb.harmonic(2.0, 5, a=1.5, b=0.25),                                          # FAST unit dom
        mcb.harmonic(1.0, 1, unit_coeffs=True, low=[-3.0], high=[8.0]),
        mcb.make_integrand(mcb.FAMILY_HARMONIC_VEC, 5, k=[1.5, -2.0, 0.25, 7.0, 3.0], a=1.25, b=0.75),
        mcb.make_integrand(mcb.FAMILY_HARMONIC_VEC, 2, k=[1.5, -2.0], a=1.0, b=1.0,
                           low=[-1, -1], high=[2, 3]),
        mcb.make_integrand(mcb.FAMILY_ABS2, 2),
        mcb.make_integrand(mcb.FAMILY_ABS2, 5, a=1.3, low=[-0.4, 0, 0, 0, 0], high=[1, 1.4, 1, 1, 1]),
        mcb.make_integrand(mcb.FAMILY_ABS3, 3, a=0.8, low=[0, -0.25, 0], high=[1, 1, 1.5]),
        mcb.make_integrand(mcb.FAMILY_ABS3, 8, a=2.0),
        mcb.harmonic(1e30, 2, a=1.0, b=1.0, unit_coeffs=False),                      # SAFE (|t| huge)
        mcb.harmonic(3.0, 2, a=float("nan"), b=1.0),                                  # SAFE, all NaN
    ]


def test_family_values_vs_oracle(gpu):
    for idx, f in enumerate(_families(gpu)):
        f.integrand_index = idx
        lo = [f.low[j] for j in range(f.dim)]
        hi = [f.high[j] for j in range(f.dim)]
        for trial, chunk, first, n in [(0, 0, 0, 2048), (3, 7, 1, 999)]:
            got = gpu.debug_eval(f, 99, trial, chunk, first, n)
            pts = _oracle.sample_uniform(lo, hi, 99, idx, trial, chunk, first, n)
            want = _oracle.eval_points(f, pts)
            nan_g, nan_w = ~np.isfinite(got), ~np.isfinite(want)
            assert np.array_equal(nan_g, nan_w), gpu.to_dsl(f)
            g, w = got[~nan_w], want[~nan_w]
            if len(w) == 0:
                continue
            if f.family in (gpu.FAMILY_ABS2, gpu.FAMILY_ABS3):
                assert np.array_equal(g, w), gpu.to_dsl(f)  # no transcendental: bit-exact
            else:
                scale = abs(f.a) + abs(f.b)
                err = np.abs(g - w).max(initial=0.0)
                # sincos within a few ulp of glibc; 1e-15 of the coefficient scale
                assert err <= 4e-15 * scale * (1 if f.k[0] < 1e6 else 1e15), (gpu.to_dsl(f), err)


# ------------------------------------------------------------------ estimator

def test_direct_mc_vs_reference_golden(gpu, golden):
    from tests.test_oracle import desc_from
    for case in golden["direct_mc"]:
        f = desc_from(case["desc"])
        st = gpu.direct_mc(f, case["seed"], case["trial"], case["chunk_base"])
        e = case["estimate"]
        row = {"value": st.value, "std_error": st.std_error, "n_samples": st.n_samples,
               "n_nonfinite": st.n_nonfinite}
        check_stats(row, fx(e["value"]), fx(e["std_error"]), e["n_samples"], e["n_nonfinite"], "direct_mc")


def test_survey_appendix_a_estimates(gpu):
    from paper_2104_10073_b200 import workloads
    fns, seed, trials = workloads.c1(1_000_000)
    out = gpu.run_direct([fns[0], fns[99]], seed, trials)
    check_stats(out[0, 0], -0.00024887253964920892, 0.0010000961624619361, 1_000_000, 0, "appendix A f001")
    assert close(out[1, 0]["value"], 0.00092141977470695628, 0.00092141977470695628, 0.00099973839472029292,
                 1_000_000, "appendix A f100")
    m, sd, _ = gpu.summarize_trials(out[0])
    assert abs(m - (-0.002062022206351116)) <= 1e-9 * 1e-3
    assert abs(sd - 0.0010213736603369853) <= 1e-6 * sd  # within the trial spread by far
    m, sd, _ = gpu.summarize_trials(out[1])
    assert abs(m - 0.00039146835923169069) <= 1e-12


def test_run_batch_vs_reference_golden(gpu, golden):
    from tests.test_oracle import desc_from
    for rb in golden["run_batch"]:
        fns = [desc_from(d) for d in rb["descs"]]
        out = gpu.run_direct(fns, rb["seed"], rb["trials"])
        for i, f in enumerate(fns):
            for t in range(rb["trials"]):
                e = rb["per_trial"][i][t]
                check_stats(out[i, t], fx(e["value"]), fx(e["std_error"]), e["n_samples"],
                            e["n_nonfinite"], "run_batch " + rb["name"])
            e0 = rb["per_trial"][i][0]
            m, sd, _ = gpu.summarize_trials(out[i])
            assert close(m, fx(rb["mean"][i]), fx(e0["value"]), fx(e0["std_error"]),
                         e0["n_samples"] - e0["n_nonfinite"], "run_batch mean")
            # stds within the reference's own trial-to-trial spread (north star), here far tighter
            assert abs(sd - fx(rb["trial_stddev"][i])) <= 1e-6 * fx(rb["trial_stddev"][i]) + 1e-15


def test_random_jobs_vs_oracle(gpu):
    """Random mixed jobs incl. partial chunks, odd dims, non-unit domains."""
    rng = np.random.default_rng(17)
    fns = []
    for i in range(40):
        fam = int(rng.integers(0, 4))
        d = int(rng.integers(3 if fam == 3 else (2 if fam == 2 else 1), 9))
        unit = bool(rng.integers(0, 2))
        lo = np.zeros(d) if unit else rng.uniform(-1, 1, d)
        hi = lo + (np.ones(d) if unit else rng.uniform(0.1, 2, d))
        fns.append(gpu.make_integrand(fam, d, k=list(rng.uniform(-6, 6, 8)), a=float(rng.uniform(-2, 2)),
                                      b=float(rng.uniform(-2, 2)), low=lo, high=hi,
                                      n_samples=int(rng.integers(2, 200_000)), index=i))
    out = gpu.run_direct(fns, 4242, 3)
    ref = _oracle.run_direct(fns, 4242, 3)
    for i, f in enumerate(fns):
        for t in range(3):
            check_stats(out[i, t], float(ref[i, t]["value"]), float(ref[i, t]["std_error"]),
                        int(ref[i, t]["n_samples"]), int(ref[i, t]["n_nonfinite"]), "random jobs vs oracle")


def test_constant_integrand_exact(gpu):
    # tests/test_estimator.cpp:44-52 and tests/test_batch.cpp:29-43
    f = gpu.harmonic(0.0, 2, a=7.0, b=3.0, low=[0, 0], high=[2, 2], n_samples=1000)
    st = gpu.direct_mc(f, 1)
    assert st.value == 28.0 and st.std_error == 0.0 and st.n_samples == 1000
    g = gpu.harmonic(0.0, 1, a=5.0, b=1.0, low=[0], high=[2], n_samples=300_000)
    out = gpu.run_direct([f, g], 1, 3)
    assert (out[0]["value"] == 28.0).all() and (out[0]["std_error"] == 0.0).all()
    assert (out[1]["value"] == 10.0).all()
    m, sd, _ = gpu.summarize_trials(out[1])
    assert m == 10.0 and sd == 0.0


def test_nonfinite_counting_and_isolation(gpu):
    # SAFE variant: |t| overflows on part of the domain -> NaN samples counted, others kept
    part = gpu.harmonic(1e308, 2, a=1.0, b=1.0, unit_coeffs=False, n_samples=100_000, index=0)
    dead = gpu.harmonic(3.0, 2, a=float("nan"), b=1.0, n_samples=1000, index=1)   # sqrt(-1-x1) analogue
    alive = gpu.make_integrand(gpu.FAMILY_ABS2, 2, n_samples=1000, index=2)
    out = gpu.run_direct([part, dead, alive], 3, 2)
    ref = _oracle.run_direct([part, dead, alive], 3, 2)
    assert np.array_equal(out["n_nonfinite"], ref["n_nonfinite"])
    assert (out[0]["n_nonfinite"] > 0).all() and (out[0]["nonfinite_warning"] == 1).all()
    assert (out[1]["status"] == gpu.TRIAL_ALL_NONFINITE).all()
    assert (out[2]["status"] == gpu.TRIAL_OK).all()
    for t in range(2):
        for i in (0, 2):
            check_stats(out[i, t], float(ref[i, t]["value"]), float(ref[i, t]["std_error"]),
                        int(ref[i, t]["n_samples"]), int(ref[i, t]["n_nonfinite"]), "non-finite vs oracle")


def test_device_list_invariance_byte_identical(gpu):
    """GPU-count invariance (multi-device analogue of acceptance.cpp:106-133).
    One physical GPU: each list entry is its own host thread + stream + shard."""
    from paper_2104_10073_b200 import workloads
    fns, seed, _ = workloads.c5(samples=70_000, n_fns=64)
    runs = [gpu.run_direct(fns, seed, 3, devices=d) for d in ([0], [0, 0], [0, 0, 0, 0], [0] * 8)]
    for r in runs[1:]:
        assert r.tobytes() == runs[0].tobytes()


def test_result_depends_only_on_seed_index_spec(gpu):
    # tests/test_batch.cpp:137-158
    a = gpu.harmonic(3.0, 2, n_samples=20_000, index=0)
    b = gpu.make_integrand(gpu.FAMILY_ABS2, 2, n_samples=20_000, index=1)
    both = gpu.run_direct([a, b], 5, 2)
    only_a = gpu.run_direct([a], 5, 2)
    assert both[0].tobytes() == only_a[0].tobytes()
    a2 = gpu.harmonic(3.0, 2, n_samples=20_000, index=1)
    moved = gpu.run_direct([a2], 5, 2)
    assert moved[0]["value"][0] != both[0]["value"][0]


def test_plan_api_matches_run_direct(gpu):
    from paper_2104_10073_b200 import workloads
    fns, seed, trials = workloads.c3(50_000)
    plan = gpu.Plan(fns, seed, trials)
    info = plan.info()
    assert info.n_fns == 100 and info.n_groups >= 2
    assert info.total_samples == 100 * 50_000 * trials
    plan.launch()
    a = plan.download()
    plan.launch()
    b = plan.download()
    assert a.tobytes() == b.tobytes()
    assert a.tobytes() == gpu.run_direct(fns, seed, trials).tobytes()
    plan.close()


def test_acceptance_c1_fig1_band(gpu):
    """acceptance.cpp:53-69 criterion 1: >= 95/100 inside 4 sigma of the closed form."""
    from paper_2104_10073_b200 import workloads
    fns, seed, trials = workloads.c1(1_000_000)
    out = gpu.run_direct(fns, seed, trials)
    passed = 0
    for n in range(1, 101):
        m, sd, _ = gpu.summarize_trials(out[n - 1])
        mse = float(np.mean(out[n - 1]["std_error"]) / math.sqrt(trials))
        band = 4.0 * max(sd, mse)
        passed += abs(m - workloads.harmonic_closed_form(workloads.harmonic_k(n))) <= band
    assert passed >= 95


def test_acceptance_c2_eq2_oracles(gpu):
    """acceptance.cpp:73-103: |x1+x2| -> 1, |x1+x2-x3| -> 7/12 within 3 std_error."""
    a = gpu.make_integrand(gpu.FAMILY_ABS2, 2, n_samples=1_000_000, index=0)
    b = gpu.make_integrand(gpu.FAMILY_ABS3, 3, n_samples=1_000_000, index=1)
    out = gpu.run_direct([a, b], 2026, 1)
    assert abs(out[0, 0]["value"] - 1.0) <= 3 * out[0, 0]["std_error"]
    assert abs(out[1, 0]["value"] - 7.0 / 12.0) <= 3 * out[1, 0]["std_error"]


@pytest.mark.gpu
def test_chunk_boundary_counts_vs_oracle(gpu):
    """Sample counts at the chunk and pair boundaries (2, odd, 65535..65537,
    2 chunks +- 1) in odd and even dimensions, one trial (trial stddev 0)."""
    fns = []
    for n in (2, 3, 65535, 65536, 65537, 131071, 131072, 131073):
        for d in (1, 3, 7, 8):
            fns.append(gpu.harmonic(3.0 + d, d, a=0.7, b=-1.3, low=[-0.5] * d, high=[0.25 + 0.1 * d] * d,
                                    n_samples=n, index=len(fns)))
    out = gpu.run_direct(fns, 31337, 1)
    ref = _oracle.run_direct(fns, 31337, 1)
    for i, f in enumerate(fns):
        check_stats(out[i, 0], float(ref[i, 0]["value"]), float(ref[i, 0]["std_error"]),
                    int(ref[i, 0]["n_samples"]), int(ref[i, 0]["n_nonfinite"]), "chunk boundaries vs oracle")
        mean, sd, n_ok = gpu.summarize_trials(out[i])
        assert n_ok == 1 and sd == 0.0 and mean == float(out[i, 0]["value"])
