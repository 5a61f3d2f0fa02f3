"""Synthetic workloads of BASELINE.json's configs.

All use seed 20200814 unless stated and integrand_index = list position, as
the reference's run_batch does (src/batch.cpp:221).

C1  make_harmonic_job(100, 1e6)   src/job_io.cpp:355-376 (Fig. 1, Eq. 1)
C2  make_harmonic_job(1000, 1e6)  the paper's 10^3-function claim
C3  mixed a_n|x1+x2| (n<50, 2-D) / b_n|x1+x2-x3| (50<=n<=100, 3-D), Eq. 2
C4  parameter scan of the 7-D harmonic over k_i = 0.01 (i+1), i < 4096
C5  10^4 integrands cycling {2-D abs, 3-D abs, harmonic d = 2..7}
"""
from __future__ import annotations

import math
from typing import List, Tuple

from . import (FAMILY_ABS2, FAMILY_ABS3, FAMILY_HARMONIC, Integrand, harmonic,
               make_integrand)

SEED = 20200814
TRIALS = 10


def harmonic_k(n: int) -> float:
    """k_n = (n + 50) / (2 pi), src/job_io.cpp:336-338."""
    return (float(n) + 50.0) / (2.0 * math.pi)


def harmonic_closed_form(k: float, dim: int = 4) -> float:
    """Re(phi^d) + Im(phi^d), phi = (e^{ik} - 1)/(ik); src/job_io.cpp:340-348 for d = 4."""
    if k == 0.0:
        return 1.0
    ik = complex(0.0, k)
    phi = (complex(math.cos(k), math.sin(k)) - 1.0) / ik
    p = phi
    for _ in range(dim - 1):
        p = p * phi
    return p.real + p.imag


def make_harmonic_job(n_count: int, samples: int, first_index: int = 0) -> List[Integrand]:
    """src/job_io.cpp:355-376: f_n = cos(k_n sum x) + sin(k_n sum x) on [0,1]^4."""
    return [harmonic(harmonic_k(n), 4, unit_coeffs=True, n_samples=samples,
                     index=first_index + n - 1) for n in range(1, n_count + 1)]


def c1(samples: int = 1_000_000) -> Tuple[List[Integrand], int, int]:
    return make_harmonic_job(100, samples), SEED, TRIALS


def c2(samples: int = 1_000_000, n_count: int = 1000, first_index: int = 0):
    return make_harmonic_job(n_count, samples, first_index), SEED, TRIALS


def c3(samples: int = 1_000_000) -> Tuple[List[Integrand], int, int]:
    """Frozen generator: a_n = 1 + 0.01 n on
    [-n/100, 1] x [0, 1 + n/100]; b_n = 1 - 0.005 n on [0,1] x [-1/4, 1] x [0, 1 + n/100]."""
    fns = []
    for n in range(1, 101):
        i = n - 1
        if n < 50:
            fns.append(make_integrand(FAMILY_ABS2, 2, a=1.0 + 0.01 * n, low=[-n / 100.0, 0.0],
                                      high=[1.0, 1.0 + n / 100.0], n_samples=samples, index=i))
        else:
            fns.append(make_integrand(FAMILY_ABS3, 3, a=1.0 - 0.005 * n,
                                      low=[0.0, -0.25, 0.0], high=[1.0, 1.0, 1.0 + n / 100.0],
                                      n_samples=samples, index=i))
    return fns, SEED, TRIALS


def c4(samples: int = 10_000_000, n_values: int = 4096, trials: int = TRIALS):
    """parameter_scan (src/batch.cpp:335-367) of the 7-D harmonic over k."""
    fns = [harmonic(0.01 * (i + 1), 7, unit_coeffs=True, n_samples=samples, index=i)
           for i in range(n_values)]
    return fns, SEED, trials


def c5(samples: int = 10_000_000, n_fns: int = 10_000, first_index: int = 0):
    """Cycle {abs2 2-D, abs3 3-D, harmonic d=2..7}; k and a vary with n."""
    fns = []
    for n in range(n_fns):
        idx = first_index + n
        kind = n % 8
        if kind == 0:
            fns.append(make_integrand(FAMILY_ABS2, 2, a=1.0 + 1e-4 * n, n_samples=samples, index=idx))
        elif kind == 1:
            fns.append(make_integrand(FAMILY_ABS3, 3, a=1.0 + 1e-4 * n, n_samples=samples, index=idx))
        else:
            d = kind  # 2..7
            fns.append(harmonic(harmonic_k(1 + n % 100), d, unit_coeffs=True, n_samples=samples,
                                index=idx))
    return fns, SEED, TRIALS
