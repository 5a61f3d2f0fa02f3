"""Config-scale parity: the GPU path (C-ABI mcb_run_direct) against the
reference's own direct_mc (src/estimator.cpp:75-92) at the sample counts of
BASELINE.json configs[3] / configs[4] — 1e7 samples per (integrand, trial),
i.e. 153 chunk partials merged in ascending order (estimator.cpp:20-34,55-73):

  * C4 subset: the 7-D harmonic scan k_i = 0.01 (i+1) at 8 scan positions
    i = 0 .. 4095 (k = 0.01 .. 40.96; small k = a nearly constant integrand);
  * C5 subset: 16 integrands cycling all 8 kinds (abs2, abs3, harmonic d=2..7);
  * threshold cases: harmonic integrands whose argument sweeps only 0.05-0.1
    rad at an extremum of a cos + b sin (var/mean^2 ~ 1e-7 .. 1e-10), where
    an unshifted sum f^2 - (sum f)^2/n would lose std_error beyond 1e-9.

Goldens: tests/golden/make_golden.py "config_scale" (reference compiled from
/root/reference/proj).  Bars: tests/_deviation.py (value 1e-9 relative with a
1e-12 V RMS(f) floor, std_error 1e-9 relative, counts identical).
"""
import json
import os

import pytest

from tests._deviation import DEVIATIONS, check_stats
from tests.test_oracle import desc_from

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.json")


def fx(h):
    return float.fromhex(h)


@pytest.fixture(scope="module")
def cases():
    with open(GOLDEN) as fh:
        return json.load(fh)["config_scale"]


def _run_group(gpu, cases, group):
    sel = [c for c in cases["cases"] if c["group"] == group]
    assert sel, group
    seed = sel[0]["seed"]
    assert all(c["seed"] == seed for c in sel)
    fns = [desc_from(c["desc"]) for c in sel]
    out = gpu.run_direct(fns, seed, cases["trials"], devices=[0])
    for i, c in enumerate(sel):
        for t, e in enumerate(c["per_trial"]):
            check_stats(out[i, t], fx(e["value"]), fx(e["std_error"]), e["n_samples"], e["n_nonfinite"],
                        f"config scale {group}")
    return sel, out


def test_c4_subset_1e7_vs_reference(gpu, cases):
    sel, out = _run_group(gpu, cases, "c4")
    assert len(sel) == 8 and all(c["desc"]["n_samples"] == 10_000_000 for c in sel)
    assert sorted(c["desc"]["integrand_index"] for c in sel) == [0, 4, 19, 99, 511, 1023, 2047, 4095]


def test_c5_subset_1e7_vs_reference(gpu, cases):
    sel, out = _run_group(gpu, cases, "c5")
    assert len(sel) == 16
    assert sorted(c["desc"]["integrand_index"] % 8 for c in sel) == sorted(list(range(8)) * 2)


def test_near_constant_threshold_cases_vs_reference(gpu, cases):
    sel, out = _run_group(gpu, cases, "threshold")
    assert len(sel) >= 8
    # the std_error bar is the point of these cases
    assert DEVIATIONS["config scale threshold std_error"][1] == 2 * len(sel)
