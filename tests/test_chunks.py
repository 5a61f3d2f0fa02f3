"""The per-chunk layer of the reference's estimator API on the GPU:
accumulate_chunk (ref include/mcbatch/estimator.hpp:70-74, src/estimator.cpp:
36-49), ChunkAccum add/merge (:9-34), reduce_chunks (:55-73) and the
UniformStream draw order (include/mcbatch/sampling.hpp:46-65,
src/sampling.cpp:78-100), through the C-ABI (mcb_accumulate_chunk) and the
source-compatible C++ headers (include/mcbatch/*.hpp).

Bars: n and n_nonfinite identical to the oracle's Welford pass; mean within
1e-12 of the chunk's RMS(f) (the GPU forms it from shifted sums instead of the
running recurrence); m2 within 1e-9 relative (floor 1e-12 n RMS(f)^2); draws
bit-exact.  CPU tests: the C++ program compiles against the headers."""
import math
import os
import subprocess

import numpy as np
import pytest

from tests import _oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "_build", "test_compat_chunks")


def _cases(gpu):
    rng = np.random.default_rng(2024)
    fns = []
    counts = [1, 2, 3, 7, 4096, 65535, 65536, 12345, 33333, 65536, 50001, 2, 65536, 999]
    for i, count in enumerate(counts):
        fam = i % 4
        d = [1, 2, 3, 4, 5, 6, 7, 8][i % 8]
        d = max(d, 2 if fam == 2 else (3 if fam == 3 else 1))
        unit = i % 3 == 0
        lo = np.zeros(d) if unit else rng.uniform(-1, 1, d)
        hi = lo + (np.ones(d) if unit else rng.uniform(0.1, 2, d))
        f = gpu.make_integrand(fam, d, k=list(rng.uniform(-9, 9, 8)), a=float(rng.uniform(-2, 2)),
                               b=float(rng.uniform(-2, 2)), low=lo, high=hi, n_samples=count,
                               index=int(rng.integers(0, 2**32)))
        fns.append((f, count, int(rng.integers(0, 50)), int(rng.integers(0, 2**32))))
    return fns


def _check_accum(got, want, label):
    assert (got.n, got.n_nonfinite) == (want.n, want.n_nonfinite), label
    if want.n == 0:
        return
    rms = math.sqrt(want.mean * want.mean + want.m2 / want.n)
    assert abs(got.mean - want.mean) <= 1e-12 * max(rms, 1e-300), (label, got.mean, want.mean)
    assert abs(got.m2 - want.m2) <= max(1e-9 * want.m2, 1e-12 * want.n * rms * rms), (label, got.m2, want.m2)


@pytest.mark.gpu
def test_accumulate_chunk_vs_oracle(gpu, oracle):
    for f, count, trial, chunk in _cases(gpu):
        got = gpu.accumulate_chunk(f, 77, trial, chunk, count)
        want = _oracle.ChunkAccum()
        assert oracle.orc_accumulate_chunk(f, 77, trial, chunk, count, want) == 0
        _check_accum(got, want, (f.family, f.dim, count))


@pytest.mark.gpu
def test_accumulate_chunk_edges(gpu, mcb):
    f = gpu.harmonic(3.0, 2, n_samples=10)
    z = gpu.accumulate_chunk(f, 1, 0, 0, 0)
    assert (z.n, z.n_nonfinite, z.mean, z.m2) == (0, 0, 0.0, 0.0)
    with pytest.raises(mcb.McbError):
        gpu.accumulate_chunk(f, 1, 0, 0, 65537)
    with pytest.raises(mcb.McbError):
        gpu.accumulate_chunk(f, 1, 0, 2**32, 10)
    # a constant integrand: exactly its value, zero spread
    c = gpu.harmonic(0.0, 3, a=2.5, b=4.0, n_samples=10)
    a = gpu.accumulate_chunk(c, 5, 1, 3, 40000)
    assert (a.n, a.mean, a.m2) == (40000, 2.5, 0.0)
    # non-finite samples are counted, not accumulated (SAFE path: 1/x at x = 0 is not hit by
    # the sampler, so use a program whose value is NaN on half the domain)
    p = gpu.Program("sqrt(x1 - 0.5)", 1)
    g = p.integrand(n_samples=10)
    b = gpu.accumulate_chunk(g, 9, 0, 0, 20000)
    assert b.n + b.n_nonfinite == 20000 and 9000 < b.n_nonfinite < 11000


@pytest.mark.gpu
def test_chunks_reduce_to_direct_mc(gpu, oracle):
    """accumulate_chunk over every chunk of an integrand + reduce_chunks (the
    reference's direct_mc decomposition, src/estimator.cpp:75-92) agrees with the
    fused direct_mc."""
    f = gpu.harmonic(7.5, 4, a=1.3, b=-0.4, low=[0, -1, 0.5, 0], high=[1, 1, 2, 0.25], n_samples=300_001,
                     index=12)
    n_chunks = (f.n_samples + 65535) // 65536
    acc = [gpu.accumulate_chunk(f, 99, 2, 5 + c, min(65536, f.n_samples - c * 65536)) for c in range(n_chunks)]
    total = _oracle.ChunkAccum()
    for a in acc:
        oracle.orc_accum_merge(total, _oracle.ChunkAccum(a.n, a.n_nonfinite, a.mean, a.m2))
    vol = gpu.volume(f)
    st = gpu.direct_mc(f, 99, 2, 5)
    assert total.n == st.n_samples
    assert abs(vol * total.mean - st.value) <= 1e-12 * abs(st.value) + 1e-15
    se = vol * math.sqrt(total.m2 / (total.n - 1) / total.n)
    assert abs(se - st.std_error) <= 1e-9 * st.std_error


def _build():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    libdir = os.path.join(ROOT, "paper_2104_10073_b200")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_compat_chunks.cpp"),
                    os.path.join(libdir, "libmcb.so"), "-Wl,-rpath," + libdir, "-o", EXE], check=True)
    return EXE


def test_compat_chunk_layer_compiles():
    assert os.path.exists(_build())


@pytest.mark.gpu
def test_compat_chunk_layer_on_gpu(gpu, oracle):
    """mcbatch::UniformStream draws, accumulate_chunk / reduce_chunks and the
    host ChunkAccum recurrences through the source-compatible headers."""
    r = subprocess.run([_build()], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = dict(line.split(" ", 1) for line in r.stdout.strip().splitlines())
    # UniformStream: 10000 draws of key {123456789, 7, 3, 11} == 1-D unit points of that key
    draws = np.array([float.fromhex(x) for x in lines["draws"].split()])
    want = _oracle.sample_uniform([0.0], [1.0], 123456789, 7, 3, 11, 0, len(draws)).ravel()
    assert np.array_equal(draws.view(np.uint64), want.view(np.uint64))
    # host ChunkAccum::add over those draws == the oracle's Welford, bit for bit
    w = _oracle.ChunkAccum()
    for x in want:
        oracle.orc_accum_add(w, float(x))
    n, nn, mean, m2 = lines["welford"].split()
    assert (int(n), int(nn)) == (w.n, w.n_nonfinite)
    assert float.fromhex(mean) == w.mean and float.fromhex(m2) == w.m2
    # accumulate_chunk of "abs(x1+x2-x3)" on [0,1]^3, chunk 4 of key {5, 2, 1, 4}, count 30000
    n, nn, mean, m2 = lines["chunk"].split()
    f = gpu.make_integrand(gpu.FAMILY_ABS3, 3, a=1.0, b=1.0, n_samples=30000, index=2)
    ref = _oracle.ChunkAccum()
    assert oracle.orc_accumulate_chunk(f, 5, 1, 4, 30000, ref) == 0
    got = _oracle.ChunkAccum(int(n), int(nn), float.fromhex(mean), float.fromhex(m2))
    _check_accum(got, ref, "compat accumulate_chunk")
    assert lines["reduce"].split()[0] == "ok"
