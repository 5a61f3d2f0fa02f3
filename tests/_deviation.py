"""Tolerances of the GPU-vs-reference parity tests, and a record of how close
each comparison came to its bar.

value:      |gpu - ref| <= max(1e-9 |ref|, 1e-12 V RMS(f))
std_error:  |gpu - ref| <= 1e-9 ref                           (§8(c) (iii))

V RMS(f) is taken from the reference's own estimate of the same (integrand,
trial): value = V mean and std_error = V sd / sqrt(n), so
(V RMS(f))^2 = V^2 (mean^2 + sd^2) = value^2 + std_error^2 n.

Every comparison records |gpu - ref| / tolerance under a label; conftest's
terminal summary prints the largest ratio per label, so a run shows the
margin, not just pass/fail.
"""
from __future__ import annotations

import math
from collections import defaultdict

REL = 1e-9
FLOOR = 1e-12

# label -> [max ratio, comparisons, detail of the max]
DEVIATIONS: dict = defaultdict(lambda: [0.0, 0, ""])


def record(label: str, ratio: float, detail: str = "") -> None:
    d = DEVIATIONS[label]
    d[1] += 1
    if ratio > d[0] or d[1] == 1:
        d[0], d[2] = max(ratio, d[0]), detail


def rms_scale(ref_value: float, ref_se: float, n_finite: int) -> float:
    """V * RMS(f) from the reference's estimate."""
    se2n = ref_se * ref_se * n_finite if math.isfinite(ref_se) else 0.0
    return math.sqrt(ref_value * ref_value + se2n)


def close(got: float, want: float, ref_value: float, ref_se: float, n_finite: int, label: str = "") -> bool:
    tol = max(REL * abs(want), FLOOR * rms_scale(ref_value, ref_se, n_finite))
    err = abs(float(got) - want)
    if tol == 0.0:
        ok = err == 0.0
        record(label + " value", 0.0 if ok else math.inf, f"got {got!r} want {want!r}")
        return ok
    record(label + " value", err / tol, f"got {got!r} want {want!r}")
    return err <= tol


def close_rel(got: float, want: float, label: str = "") -> bool:
    tol = REL * abs(want)
    err = abs(float(got) - want)
    if tol == 0.0:
        ok = err == 0.0
        record(label + " std_error", 0.0 if ok else math.inf, f"got {got!r} want {want!r}")
        return ok
    record(label + " std_error", err / tol, f"got {got!r} want {want!r}")
    return err <= tol


def check_stats(row, want_value: float, want_se: float, want_n: int, want_nn: int, label: str = "") -> None:
    """One (integrand, trial) McEstimate against the reference's."""
    assert int(row["n_samples"]) == want_n, (label, int(row["n_samples"]), want_n)
    assert int(row["n_nonfinite"]) == want_nn, (label, int(row["n_nonfinite"]), want_nn)
    got_v, got_se = float(row["value"]), float(row["std_error"])
    assert close(got_v, want_value, want_value, want_se, want_n - want_nn, label), (label, got_v, want_value)
    if math.isinf(want_se):
        assert math.isinf(got_se), (label, got_se)
    else:
        assert close_rel(got_se, want_se, label), (label, got_se, want_se)


def summary_lines() -> list:
    out = []
    for label in sorted(DEVIATIONS):
        mx, n, detail = DEVIATIONS[label]
        out.append(f"{label:55s} {n:6d} comparisons, max |dev|/tol = {mx:.3g}  ({detail})")
    return out
