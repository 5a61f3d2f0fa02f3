"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/mcb/mcb.h declares, and its host-side helpers keep the
reference's contracts (validate wording src/batch.cpp:62-120, key derivation
src/sampling.cpp:84-87, volume src/sampling.cpp:16-20, summarize_trials
src/estimator.cpp:320-337).  Compute entry points must fail loudly without a
device — there is no CPU fallback."""
import ctypes
import os
import re

import numpy as np
import pytest

from tests import _oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "mcb", "mcb.h")).read()
    return sorted(set(re.findall(r"MCB_API\s+[\w\s\*]+?\b(mcb_\w+)\s*\(", src)))


def test_exports_every_declared_symbol(mcb):
    decl = declared_symbols()
    assert len(decl) >= 19
    assert sorted(mcb.ABI_SYMBOLS) == decl
    out = os.popen(f"nm -D --defined-only {mcb.LIB_PATH}").read()
    exported = set(re.findall(r" T (mcb_\w+)", out))
    assert set(decl) <= exported, set(decl) - exported
    assert mcb.lib.mcb_abi_version() == 2


def test_library_is_native_sm100a(mcb):
    out = os.popen(f"cuobjdump -lelf {mcb.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out


def test_stream_key_matches_oracle(mcb):
    rng = np.random.default_rng(1)
    for _ in range(200):
        seed, idx = int(rng.integers(0, 2**64, dtype=np.uint64)), int(rng.integers(0, 2**32))
        assert mcb.stream_key(seed, idx) == _oracle.stream_key(seed, idx)


def test_to_dsl_exact_reference_sources(mcb):
    f = mcb.harmonic(1.0, 4, unit_coeffs=True)
    assert mcb.to_dsl(f) == "cos(k*(x1+x2+x3+x4)) + sin(k*(x1+x2+x3+x4))"  # src/job_io.cpp:367
    f = mcb.harmonic(1.0, 2, a=2.0, b=3.0)
    assert mcb.to_dsl(f) == "a*cos(k*(x1+x2)) + b*sin(k*(x1+x2))"
    f = mcb.make_integrand(mcb.FAMILY_HARMONIC_VEC, 3, k=[1, 2, 3], a=1.0, b=1.0)
    assert mcb.to_dsl(f) == "a*cos(k1*x1+k2*x2+k3*x3) + b*sin(k1*x1+k2*x2+k3*x3)"
    assert mcb.to_dsl(mcb.make_integrand(mcb.FAMILY_ABS2, 2)) == "abs(x1+x2)"  # test_batch.cpp:49
    assert mcb.to_dsl(mcb.make_integrand(mcb.FAMILY_ABS3, 3)) == "abs(x1+x2-x3)"
    assert mcb.to_dsl(mcb.make_integrand(mcb.FAMILY_ABS3, 3, a=0.5)) == "a*abs(x1+x2-x3)"


def test_volume_left_to_right(mcb):
    f = mcb.make_integrand(mcb.FAMILY_ABS3, 3, low=[0.1, -0.25, 0.3], high=[1.7, 1.0, 2.9])
    assert mcb.volume(f) == _oracle.load().orc_volume(ctypes.byref(f))


def test_validate_reports_every_violation(mcb):
    # mirrors tests/test_batch.cpp:60-89 for the family descriptors
    good = mcb.harmonic(2.0, 2, n_samples=1000)
    bad_dim = mcb.make_integrand(mcb.FAMILY_ABS3, 2, n_samples=1000)
    bad_dom = mcb.harmonic(2.0, 2, low=[0, 1], high=[1, 1], n_samples=1000)
    bad_n = mcb.harmonic(2.0, 1, n_samples=1)
    v = mcb.validate([good, bad_dim, bad_dom, bad_n, good], 2, names=["a", "b", "c", "d", "a"])
    msgs = {(i, m) for i, m in v}
    assert (1, "x3 exceeds dim=2") in msgs
    assert (2, "domain is invalid (need low[i] < high[i], finite, dim >= 1)") in msgs
    assert (3, "samples must be >= 2") in msgs
    assert any("duplicate integrand name (2 occurrences)" in m for _, m in v)
    assert mcb.validate([good], 2) == []
    assert (-1, "trials must be >= 1") in mcb.validate([good], 0)
    assert (-1, "integrand list is empty") in mcb.validate([], 1)


def test_partition_lpt_balances_and_is_deterministic(mcb):
    from paper_2104_10073_b200 import workloads
    fns, _, _ = workloads.c5(samples=1_000_000, n_fns=1000)
    for shards in (1, 2, 4, 8):
        s = mcb.partition(fns, 10, shards)
        assert set(s.tolist()) == set(range(shards))
        assert np.array_equal(s, mcb.partition(fns, 10, shards))
        loads = np.bincount(s, minlength=shards)
        assert loads.max() - loads.min() <= max(2, len(fns) // shards // 5)


def test_summarize_trials_matches_oracle(mcb, oracle):
    rng = np.random.default_rng(3)
    per = np.zeros(10, dtype=mcb.TRIAL_DTYPE)
    per["value"] = rng.normal(size=10)
    per["status"][3] = mcb.TRIAL_ALL_NONFINITE
    m, sd, nok = mcb.summarize_trials(per)
    mo, sdo, nko = ctypes.c_double(), ctypes.c_double(), ctypes.c_uint32()
    oracle.orc_summarize_trials(per.ctypes.data_as(ctypes.POINTER(mcb.TrialStats)), 10,
                                ctypes.byref(mo), ctypes.byref(sdo), ctypes.byref(nko))
    assert (m, sd, nok) == (mo.value, sdo.value, nko.value) and nok == 9


def test_compute_without_device_fails_loudly(mcb):
    if mcb.device_count() > 0:
        pytest.skip("a GPU is visible; covered by the gpu tests")
    f = mcb.harmonic(2.0, 2, n_samples=1000)
    with pytest.raises(mcb.McbError) as e:
        mcb.run_direct([f], 1, 2)
    assert e.value.status == 4  # MCB_ERR_NO_DEVICE
    with pytest.raises(mcb.McbError):
        mcb.debug_points(1, 0, 0, 0, 0, 4, [0.0], [1.0])


def test_accumulate_chunk_argument_errors(mcb):
    """mcb_accumulate_chunk rejects bad arguments before touching a device
    (count above the chunk size, a chunk index past 32 bits, an invalid
    descriptor); a zero count is an empty accumulator on any machine."""
    f = mcb.harmonic(2.0, 2, n_samples=10)
    for args in ((1, 0, 0, 65537), (1, 0, 2**32, 10)):
        with pytest.raises(mcb.McbError) as e:
            mcb.accumulate_chunk(f, *args)
        assert e.value.status in (1, 5), str(e.value)  # invalid argument / out of range
    bad = mcb.harmonic(2.0, 2, low=[0.0, 1.0], high=[1.0, 0.5], n_samples=10)
    with pytest.raises(mcb.McbError) as e:
        mcb.accumulate_chunk(bad, 1, 0, 0, 100)
    assert e.value.status == 2 and "domain is invalid" in str(e.value)
    z = mcb.accumulate_chunk(f, 1, 0, 0, 0)
    assert (z.n, z.n_nonfinite, z.mean, z.m2) == (0, 0, 0.0, 0.0)
    if mcb.device_count() == 0:
        with pytest.raises(mcb.McbError) as e:
            mcb.accumulate_chunk(f, 1, 0, 0, 100)
        assert e.value.status == 4  # MCB_ERR_NO_DEVICE: no CPU fallback


def test_validation_error_precedes_device_check(mcb):
    with pytest.raises(mcb.McbError) as e:
        mcb.run_direct([mcb.harmonic(2.0, 2, n_samples=1)], 1, 2)
    assert e.value.status == 2 and "samples must be >= 2" in str(e.value)


def test_validate_edges(mcb):
    """Sizes and descriptors at and past the supported limits."""
    f9 = mcb.harmonic(1.0, 8, n_samples=100)
    f9.dim = 9
    assert (0, "dim 9 exceeds the supported maximum 8") in mcb.validate([f9], 1)
    f0 = mcb.harmonic(1.0, 1, n_samples=100)
    f0.dim = 0
    assert (0, "dim must be >= 1") in mcb.validate([f0], 1)
    huge = mcb.harmonic(1.0, 2, n_samples=(2**32 + 1) * 65536)
    assert (0, "samples exceed 2^32 chunks (chunk_index is 32-bit)") in mcb.validate([huge], 1)
    many = mcb.harmonic(1.0, 2, n_samples=2**20 * 65536)
    assert (0, "chunks x trials exceeds 2^32 work units for one integrand") in mcb.validate([many], 2**13)
    nan_dom = mcb.harmonic(1.0, 2, low=[0.0, float("nan")], high=[1.0, 1.0], n_samples=100)
    inf_dom = mcb.harmonic(1.0, 2, low=[0.0, 0.0], high=[1.0, float("inf")], n_samples=100)
    msg = "domain is invalid (need low[i] < high[i], finite, dim >= 1)"
    assert (0, msg) in mcb.validate([nan_dom], 1) and (0, msg) in mcb.validate([inf_dom], 1)
    fam = mcb.harmonic(1.0, 2, n_samples=100)
    fam.family = 9
    assert (0, "unknown integrand family 9") in mcb.validate([fam], 1)
    flg = mcb.harmonic(1.0, 2, n_samples=100)
    flg.flags |= 0x80
    assert (0, "unknown flag bits") in mcb.validate([flg], 1)
    unit = mcb.harmonic(1.0, 2, a=2.0, b=1.0, n_samples=100)
    unit.flags = mcb.FLAG_UNIT_COEFFS
    assert (0, "unit-coefficient flag needs the harmonic family with a = b = 1") in mcb.validate([unit], 1)
    prog = mcb.make_integrand(mcb.FAMILY_PROGRAM, 2, n_samples=100)
    assert (0, "program family needs a compiled program") in mcb.validate([prog], 1)
    assert mcb.validate([mcb.harmonic(1.0, 8, n_samples=2)], 1) == []  # the minimum budget
