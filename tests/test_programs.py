"""Arbitrary DSL integrands (MCB_FAMILY_PROGRAM): the
GPU postfix interpreter against the reference.

CPU tests pin the pure-Python DSL oracle (tests/_dsl_oracle.py) bit-exactly to
values and estimates produced by the reference itself (golden "programs"),
and check the host compiler's contract (errors in the reference's wording,
stack depth / instruction counts).  GPU tests compare the interpreter with
the golden values and with the oracle.

Tolerances: per-sample values |gpu - ref| <= 1e-12 * max(1, |ref|) with the
same non-finite pattern (libdevice transcendentals are within 2 ulp of
glibc); estimates 1e-9 relative (floor 1e-12 of the per-sample scale);
n_samples / n_nonfinite identical."""
import json
import math
import os

import numpy as np
import pytest

from tests import _dsl_oracle as dsl
from tests import _oracle
from tests._deviation import check_stats

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.json")


def fx(h):
    return float.fromhex(h)


@pytest.fixture(scope="module")
def progs():
    with open(GOLDEN) as fh:
        return json.load(fh)["programs"]


def _case(c):
    params = {k: fx(v) for k, v in c["params"].items()}
    lo = [fx(x) for x in c["low"]]
    hi = [fx(x) for x in c["high"]]
    return params, lo, hi


# ------------------------------------------------------------------ CPU

def test_oracle_values_match_reference(progs, oracle):
    for c in progs:
        params, lo, hi = _case(c)
        p = dsl.Program(c["source"], c["dim"], params)
        pts = _oracle.sample_uniform(lo, hi, c["seed"], c["index"], c["trial"], c["chunk_base"], 0, 64)
        got = np.array([p(row) for row in pts])
        want = np.array([fx(v) for v in c["values"]])
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)) or \
            np.allclose(got, want, rtol=0, atol=0, equal_nan=True), c["source"]


def test_oracle_estimates_match_reference(progs, oracle):
    for c in progs:
        if c["n_samples"] > 100_000:
            continue  # pure-Python Welford: keep the CPU suite fast
        params, lo, hi = _case(c)
        p = dsl.Program(c["source"], c["dim"], params)
        n, chunks, rem = c["n_samples"], [], c["n_samples"]
        ch = 0
        while rem > 0:
            cnt = min(65536, rem)
            pts = _oracle.sample_uniform(lo, hi, c["seed"], c["index"], c["trial"], c["chunk_base"] + ch, 0, cnt)
            chunks.append([p(row) for row in pts])
            rem -= cnt
            ch += 1
        vol = 1.0
        for a, b in zip(lo, hi):
            vol *= b - a
        res = dsl.welford_direct_mc(chunks, vol)
        e = c["estimate"]
        if e["status"] == 1:
            assert res is None
            continue
        assert res[0] == fx(e["value"]) and res[1] == fx(e["std_error"]), c["source"]
        assert (res[2], res[3]) == (e["n_samples"], e["n_nonfinite"])


def test_compiler_contract(mcb):
    p = mcb.Program("cos(k*(x1+x2+x3+x4)) + sin(k*(x1+x2+x3+x4))", 4, ["k"])
    # reference postfix: 21 instructions, stack 4; the GPU
    # form shares k*(x1+..+x4), folds loads
    # into operands and fuses cos(E) + sin(E): Add, Add, Add, Mul, CosPlusSin in 1 slot
    assert len(dsl.Program(p.source, 4, {"k": 1.0}).code) == 21
    assert (p.n_instr, p.depth) == (5, 1)
    assert mcb.Program("a*x1 + b + c", 1, ["c", "a", "b"]).param_names == ["a", "b", "c"]
    # squares compile to one multiply of the shared operand (x1-c computed once):
    # Sub, Mul, Sub, Mul, Add, Mul(-100), Exp; cubes and fourth powers to two
    # multiplies, E^-1 to a division, E^1 / E^0 to E / 1; other exponents stay pow
    peak = mcb.Program("exp(-100*((x1-c)^2+(x2-c)^2))", 2, ["c"])
    assert (peak.n_instr, peak.depth) == (7, 2)
    assert mcb.Program("pow(x1-c, 2)", 1, ["c"]).n_instr == 2
    assert mcb.Program("(x1-c)^3", 1, ["c"]).n_instr == 3
    assert mcb.Program("(x1-c)^4", 1, ["c"]).n_instr == 3
    assert mcb.Program("(x1-c)^2.5", 1, ["c"]).n_instr == 2
    assert mcb.Program("x1^-1 + x1^0 + x1^1", 1).n_instr == 3  # Div, Add(+1 folded), Add
    # operations on constants only are folded by the host's libm (the reference's values)
    assert mcb.Program("sin(1)*x1 + 2^0.5 + exp(-2)", 1).n_instr == 3  # Mul, Add, Add (never reassociated)
    cases = {
        "x3": "x3 exceeds dim=2",
        "2+": "expression does not parse: expected a number, identifier or '(' (at offset 2)",
        "q*x1": "unbound parameter 'q'",
        "sin(x1,x2)": "function 'sin' expects 1 argument(s), got 2",
        "foo(x1)": "unknown function 'foo'",
        "sin": "expected '(' after function name 'sin'",
        "1.5e": "unexpected trailing input",
        "(x1": "expected ')'",
        "x1 $ 2": "unexpected character '$'",
        "": "empty expression",
    }
    for src, msg in cases.items():
        with pytest.raises(mcb.McbError) as e:
            mcb.Program(src, 2, ["a"])
        assert e.value.status == 2 and msg in str(e.value), (src, str(e.value))
    # deep right-nested expressions: the deeper operand is evaluated first
    # (Sethi-Ullman), so a chain of 20 levels still needs 2 slots (the
    # reference's stack machine needs 21)
    deep = "".join(f"sin(x1*{i}+" for i in range(1, 21)) + "x1" + ")" * 20
    assert mcb.Program(deep, 1).depth <= 2
    wide = "+".join(f"sin({i}*x1)*cos({i}*x1)" for i in range(1, 30))
    assert mcb.Program(wide, 1).depth <= 4
    nested = "x1"
    for i in range(1, 20):
        nested = f"x1*(sin({i}*x1)+{nested})"
    assert mcb.Program(nested, 1).depth <= 3


def test_grammar_matches_oracle_parser(mcb):
    """Precedence / associativity (ref tests/test_expr.cpp:30-42, 144-227):
    the C++ compiler and the independent Python parser agree on values."""
    rng = np.random.default_rng(424242)
    ops = "+-*/^"
    for _ in range(300):
        src = ""
        for t in range(int(rng.integers(1, 7))):
            if t:
                src += ops[int(rng.integers(0, 5))]
            src += "-" * int(rng.integers(0, 3))
            src += ["2", "3", "x1", "a", "0.5"][int(rng.integers(0, 5))]
        p = dsl.Program(src, 1, {"a": 1.7})
        q = mcb.Program(src, 1, ["a"])
        assert 1 <= q.n_instr <= len(p.code), src
    for src, val in [("2+3*4", 14.0), ("2^3^2", 512.0), ("-2^2", 4.0), ("2^-1", 0.5), ("8/4/2", 1.0),
                     ("2-3-4", -5.0)]:
        assert dsl.Program(src, 1, {})([0.0]) == val


def test_validate_reports_program_errors(mcb):
    p_ok = mcb.Program("x1*a", 1, ["a"])
    f = p_ok.integrand({"a": 2.0}, n_samples=1000)
    assert mcb.validate([f], 2) == []
    g = mcb.make_integrand(mcb.FAMILY_PROGRAM, 1, n_samples=1000)
    assert any("program family needs a compiled program" in m for _, m in mcb.validate([g], 2))
    h = p_ok.integrand({"a": 2.0}, n_samples=1000)
    h.dim = 2
    h.low[1], h.high[1] = 0.0, 1.0
    assert any("compiled for dim=1" in m for _, m in mcb.validate([h], 2))


# ------------------------------------------------------------------ GPU

def _values_close(got, want):
    bad_g, bad_w = ~np.isfinite(got), ~np.isfinite(want)
    assert np.array_equal(bad_g, bad_w)
    g, w = got[~bad_w], want[~bad_w]
    return np.all(np.abs(g - w) <= 1e-12 * np.maximum(1.0, np.abs(w)))


@pytest.mark.gpu
def test_interpreter_values_match_reference(gpu, progs):
    for c in progs:
        params, lo, hi = _case(c)
        p = gpu.Program(c["source"], c["dim"], list(params))
        f = p.integrand(params, low=lo, high=hi, n_samples=c["n_samples"], index=c["index"])
        got = gpu.debug_eval(f, c["seed"], c["trial"], c["chunk_base"], 0, 64)
        want = np.array([fx(v) for v in c["values"]])
        assert _values_close(got, want), c["source"]
        # odd offsets inside the chunk (pair straddling)
        got2 = gpu.debug_eval(f, c["seed"], c["trial"], c["chunk_base"], 3, 61)
        assert _values_close(got2, want[3:]), c["source"]


@pytest.mark.gpu
def test_eval_points_match_reference(gpu, progs):
    """Program.evaluate (mcb_program_eval_points, the interpreter at given
    points: the mcbatch::CompiledProgram::evaluate path) on the reference's
    own sample points reproduces its values."""
    for c in progs:
        params, lo, hi = _case(c)
        p = gpu.Program(c["source"], c["dim"], list(params))
        pts = gpu.debug_points(c["seed"], c["index"], c["trial"], c["chunk_base"], 0, 64, lo, hi)
        got = p.evaluate(pts, params)
        want = np.array([fx(v) for v in c["values"]])
        assert _values_close(got, want), c["source"]
        # and exactly what the sampling kernels evaluate at those points
        f = p.integrand(params, low=lo, high=hi, n_samples=c["n_samples"], index=c["index"])
        ker = gpu.debug_eval(f, c["seed"], c["trial"], c["chunk_base"], 0, 64)
        assert np.array_equal(np.isfinite(got), np.isfinite(ker)), c["source"]
        fin = np.isfinite(ker)
        assert np.array_equal(got[fin].view(np.uint64), ker[fin].view(np.uint64)), c["source"]


@pytest.mark.gpu
def test_squares_and_constant_folding_exact(gpu):
    """E^2 / pow(E, 2) run as E*E (E^3, E^4 as two multiplies, E^-1 as 1/E)
    and constant sub-expressions are folded on the host with its libm (the
    library the reference evaluates them with): the GPU values equal the same
    operations in numpy bit for bit, specials included; and the cubes and
    fourth powers stay within 2 ulp of glibc's pow."""
    rng = np.random.default_rng(5)
    x = np.concatenate([rng.uniform(-3, 3, 200), [0.0, -0.0, 1e200, -1e200, 1e-170, np.inf, -np.inf, np.nan]])
    pts = x.reshape(-1, 1)
    c = 0.3125
    cases = [("(x1-c)^2", lambda v: (v - c) * (v - c)),
             ("pow(x1-c, 2)", lambda v: (v - c) * (v - c)),
             ("2*pi*x1", lambda v: (2 * math.pi) * v),
             ("-100*x1 + 1/3", lambda v: -100.0 * v + 1.0 / 3.0),
             ("x1*2*pi", lambda v: (v * 2) * math.pi),
             ("x1^-1", lambda v: 1.0 / v),
             ("x1^1 + x1^0", lambda v: v + 1.0),
             ("sin(1)*x1 + 2^0.5", lambda v: math.sin(1.0) * v + 2.0 ** 0.5),
             ("(x1-c)^4", lambda v: ((v - c) * (v - c)) * ((v - c) * (v - c))),
             ("(x1-c)^3", lambda v: ((v - c) * (v - c)) * (v - c))]
    for src, ref in cases:
        p = gpu.Program(src, 1, ["c"] if "c" in src.replace("pi", "") else [])
        got = p.evaluate(pts, {"c": c} if p.param_names else None)
        with np.errstate(all="ignore"):
            want = ref(x)
        assert np.array_equal(np.isnan(got), np.isnan(want)), src
        ok = ~np.isnan(want)
        assert np.array_equal(got[ok].view(np.uint64), want[ok].view(np.uint64)), src
    for src, e in (("(x1-c)^3", 3.0), ("(x1-c)^4", 4.0)):
        got = gpu.Program(src, 1, ["c"]).evaluate(pts, {"c": c})
        y = x - c
        fin = np.isfinite(y) & (np.abs(y) > 1e-60) & (np.abs(y) < 1e60)
        want = np.array([math.pow(float(v), e) for v in y[fin]])
        assert np.all(np.abs(got[fin] - want) <= 2 * np.spacing(np.abs(want))), src


@pytest.mark.gpu
def test_dsl_exp_accuracy(gpu):
    """The DSL's exp (dev::mcb_exp: two-term reduction, degree-13 Taylor, the
    exponent field; libdevice beyond |x| >= 708) within 2 ulp of glibc's exp on
    [-707.9, 707.9], and glibc's values for the specials, overflow and the
    subnormal range."""
    rng = np.random.default_rng(9)
    x = np.concatenate([rng.uniform(-707.9, 707.9, 20000), rng.uniform(-5, 5, 20000), rng.uniform(-1e-3, 1e-3, 5000),
                        [0.0, -0.0, 1e-300, 707.99, -707.99, 708.0, -708.0, 709.7, 709.79, 710.0, -744.0,
                         -746.0, np.inf, -np.inf, np.nan]])
    got = gpu.Program("exp(x1)", 1).evaluate(x.reshape(-1, 1))
    def glibc_exp(v):
        try:
            return math.exp(v)
        except OverflowError:
            return math.inf
    want = np.array([glibc_exp(v) for v in x])
    assert np.array_equal(np.isnan(got), np.isnan(x))
    ok = ~np.isnan(x)
    fin = ok & np.isfinite(want) & (want > 2.3e-308)
    assert np.all(np.abs(got[fin] - want[fin]) <= 2 * np.spacing(want[fin]))
    with np.errstate(invalid="ignore"):  # inf - inf where both overflowed
        assert np.all((got[ok & ~fin] == want[ok & ~fin]) | (np.abs(got[ok & ~fin] - want[ok & ~fin]) <= 5e-324))


@pytest.mark.gpu
def test_parameter_scan_failing_value_raises(gpu):
    """A scanned value whose trials all fail makes the scan throw, as in the
    reference (src/batch.cpp:320-329 success rule, :360-364 throw)."""
    p = gpu.Program("log(x1 - a)", 1, ["a"])
    out, summ = gpu.parameter_scan(p, {"a": 0.0}, "a", [0.0, -1.0], trials=3, seed=4, n_samples=2000)
    assert len(summ) == 2 and all(n == 3 for _, _, n in summ)
    with pytest.raises(RuntimeError, match=r"parameter_scan: a#1 failed: 0 of 3"):
        gpu.parameter_scan(p, {"a": 0.0}, "a", [0.0, 2.0], trials=3, seed=4, n_samples=2000)


@pytest.mark.gpu
def test_interpreter_estimates_match_reference(gpu, progs):
    for c in progs:
        params, lo, hi = _case(c)
        p = gpu.Program(c["source"], c["dim"], list(params))
        f = p.integrand(params, low=lo, high=hi, n_samples=c["n_samples"], index=c["index"])
        st = gpu.direct_mc(f, c["seed"], c["trial"], c["chunk_base"])
        e = c["estimate"]
        assert st.status == e["status"], c["source"]
        assert (st.n_samples, st.n_nonfinite) == (e["n_samples"], e["n_nonfinite"]), c["source"]
        if e["status"] != 0:
            continue
        check_stats({"value": st.value, "std_error": st.std_error, "n_samples": st.n_samples,
                     "n_nonfinite": st.n_nonfinite}, fx(e["value"]), fx(e["std_error"]), e["n_samples"],
                    e["n_nonfinite"], "programs direct_mc")


@pytest.mark.gpu
def test_program_matches_family_path(gpu):
    """The same Fig.1 integrand through the interpreter and the fused family
    kernel agree to 1e-12 per trial (different sincos implementations)."""
    from paper_2104_10073_b200 import workloads
    fam = workloads.c1(200_000)[0][:5]
    p = gpu.Program("cos(k*(x1+x2+x3+x4)) + sin(k*(x1+x2+x3+x4))", 4, ["k"])
    progs = [p.integrand({"k": f.k[0]}, n_samples=200_000, index=f.integrand_index) for f in fam]
    a = gpu.run_direct(fam, 20200814, 3)
    b = gpu.run_direct(progs, 20200814, 3)
    assert np.array_equal(a["n_samples"], b["n_samples"])
    assert np.all(np.abs(a["value"] - b["value"]) <= 1e-12)


@pytest.mark.gpu
def test_mixed_families_and_programs_device_invariant(gpu):
    from paper_2104_10073_b200 import workloads
    fns = list(workloads.c5(samples=70_000, n_fns=16)[0])
    p1 = gpu.Program("exp(-a*((x1-0.5)^2+(x2-0.5)^2))", 2, ["a"])
    p2 = gpu.Program("log(x1)*x2 + floor(4*x3)", 3)
    for i, (p, par) in enumerate([(p1, {"a": 100.0}), (p2, {}), (p1, {"a": 3.0})]):
        fns.append(p.integrand(par, low=[-1, 0, 0][:p.dim], high=[1, 1, 1][:p.dim], n_samples=90_000,
                               index=16 + i))
    runs = [gpu.run_direct(fns, 99, 3, devices=d) for d in ([0], [0, 0], [0, 0, 0])]
    assert runs[0].tobytes() == runs[1].tobytes() == runs[2].tobytes()
    # the log(x1) program on x1 in [-1, 1] has ~half non-finite samples
    assert 0.4 < runs[0][17]["n_nonfinite"][0] / 90_000 < 0.6


@pytest.mark.gpu
def test_random_programs_vs_oracle(gpu, oracle):
    from tests.golden.make_golden import random_source
    rng = np.random.default_rng(7)
    for i in range(12):
        src = random_source(rng, 3, ["a", "b"])
        params = {"a": float(rng.uniform(-2, 2)), "b": float(rng.uniform(0, 3))}
        p = dsl.Program(src, 3, params)
        q = gpu.Program(src, 3, list(params))
        n = 3000
        f = q.integrand(params, n_samples=n, index=i)
        got = gpu.debug_eval(f, 555, 1, 2, 0, n)
        pts = _oracle.sample_uniform([0.0] * 3, [1.0] * 3, 555, i, 1, 2, 0, n)
        want = np.array([p(row) for row in pts])
        assert _values_close(got, want), src


@pytest.mark.gpu
def test_cos_plus_sin_fusion(gpu):
    """cos(E) + sin(E) runs as one fused op: the table form for |E| < 2^20,
    libdevice beyond and for non-finite E.  Per-sample values within 4 ulp of 1
    (absolute) of glibc's cos + sin on both sides of the switch (k = 3 keeps E
    small, k = 1e7 crosses 2^20 inside [0, 1]), NaN where E is NaN, and the
    runtime-specialised kernel bit-identical to the interpreter."""
    n = 4000
    cases = [("cos(k*x1) + sin(k*x1)", {"k": 3.0}), ("sin(k*x1) + cos(k*x1)", {"k": 1e7}),
             ("cos(log(x1-0.5)) + sin(log(x1-0.5))", {})]
    for i, (src, params) in enumerate(cases):
        q = gpu.Program(src, 1, list(params))
        assert q.n_instr <= 3, src  # fused: no separate sincos + add
        f = q.integrand(params, n_samples=n, index=i)
        got = gpu.debug_eval(f, 31, 0, 0, 0, n)
        pts = _oracle.sample_uniform([0.0], [1.0], 31, i, 0, 0, 0, n)
        want = np.array([dsl.Program(src, 1, params)(row) for row in pts])
        bad = ~np.isfinite(want)
        assert np.array_equal(~np.isfinite(got), bad), src
        assert np.all(np.abs(got[~bad] - want[~bad]) <= 4 * 2.0 ** -52), (src, np.abs(got - want).max())
        if params.get("k") == 1e7:
            t = params["k"] * pts[:, 0]
            assert (t < 2 ** 20).any() and (t >= 2 ** 20).any()
    assert gpu.program_jit(2) == 2, gpu.program_jit_error()
    fns = [gpu.Program(src, 1, list(params)) for src, params in cases]
    ints = [p.integrand(params, n_samples=300_000, index=i) for i, (p, (_, params)) in enumerate(zip(fns, cases))]
    try:
        a = gpu.run_direct(ints, 5, 2)
        assert gpu.program_jit_error() == "", gpu.program_jit_error()
        gpu.program_jit(0)
        b = gpu.run_direct(ints, 5, 2)
    finally:
        gpu.program_jit(1)
    assert a.tobytes() == b.tobytes()


@pytest.mark.gpu
def test_jit_bit_identical_to_interpreter(gpu, progs):
    """Runtime-specialised programs (NVRTC, csrc/jit.cpp) against the bytecode
    interpreter: every per-trial McEstimate byte-identical, in all five modes
    (direct, unit cube, cells CTA-per-tile, small cells warp-per-tile, small
    cells of a large grid thread-per-cell), for
    the golden programs incl. non-finite patterns and the random ones."""
    assert gpu.program_jit(2) == 2, gpu.program_jit_error()  # always: every launch specialised
    keep, fns = [], []
    for i, c in enumerate(progs):
        params, lo, hi = _case(c)
        p = gpu.Program(c["source"], c["dim"], list(params))
        keep.append(p)
        fns.append(p.integrand(params, low=lo, high=hi, n_samples=min(c["n_samples"], 70_000), index=i))
    unit = gpu.Program("exp(-3*(x1-0.4)^2) * cos(5*x2) + x3", 3)
    keep.append(unit)
    fns.append(unit.integrand(n_samples=100_000, index=len(fns)))          # mode 1
    cells = unit.integrand(low=[-1, 0, 0], high=[1, 2, 1], n_samples=300_000, index=len(fns) + 1)
    fns.append(gpu.stratify(cells, cells_per_dim=2))                         # mode 2 (75 000 / cell)
    fns.append(gpu.stratify(unit.integrand(n_samples=200_000, index=len(fns) + 2), cells_per_dim=8))  # mode 3
    fns.append(gpu.stratify(unit.integrand(n_samples=200_000, index=len(fns) + 2)))  # mode 4: 16^3 cells
    fns.append(gpu.tree(unit.integrand(n_samples=80_000, index=len(fns) + 3), samples_per_cell=500))
    n0 = gpu.program_jit_compiles()
    a = gpu.run_direct(fns, 99, 2)
    assert gpu.program_jit_error() == "", gpu.program_jit_error()
    assert gpu.program_jit_compiles() > n0 or os.environ.get("MCB_JIT_CACHE", "") != "0"
    gpu.program_jit(0)
    try:
        b = gpu.run_direct(fns, 99, 2)
    finally:
        gpu.program_jit(1)
    for i in range(len(fns)):
        assert a[i].tobytes() == b[i].tobytes(), (i, a[i], b[i])


def test_jit_code_compiles_for_every_golden_program(mcb, progs, tmp_path, monkeypatch):
    """The generated straight-line code of every golden program (and a few
    edge cases) compiles under NVRTC for sm_100a — no device needed."""
    monkeypatch.setenv("MCB_JIT_CACHE", str(tmp_path))
    srcs = [(c["source"], c["dim"], list(c["params"])) for c in progs[:3]]
    srcs += [("7", 1, []), ("1e308*1e308 - x1", 1, []), ("a+b+c+d+e2+f+g+h", 1, list("abcdfgh") + ["e2"])]
    salt = f" + 0*x1*{os.getpid()}"  # a program no earlier test of this process compiled
    for src, dim, names in srcs:
        p = mcb.Program("(" + src + ")" + salt, dim, names)
        p.jit_build()
        assert mcb.program_jit_error() == "", (src, mcb.program_jit_error())
    assert len(list(tmp_path.iterdir())) >= 5 * len(srcs)  # five kernel modes each, cached


@pytest.mark.gpu
def test_jit_same_code_different_dimension(gpu):
    """One instruction list in two dimensions is two specialised kernels (the
    sampler's D differs): both bit-identical to the interpreter."""
    assert gpu.program_jit(2) == 2
    p1, p3 = gpu.Program("x1*x1", 1), gpu.Program("x1*x1", 3)
    fns = [p1.integrand(low=[0.0], high=[2.0], n_samples=50_000, index=0),
           p3.integrand(low=[0.0, 0.0, 0.0], high=[2.0, 1.0, 1.0], n_samples=50_000, index=0)]
    a = [gpu.run_direct([f], 5, 2) for f in fns]
    gpu.program_jit(0)
    try:
        b = [gpu.run_direct([f], 5, 2) for f in fns]
    finally:
        gpu.program_jit(1)
    for x, y in zip(a, b):
        assert x.tobytes() == y.tobytes()


@pytest.mark.gpu
def test_jit_automatic_mode(gpu, tmp_path, monkeypatch):
    """Default mode: a small one-shot run of an uncached program interprets
    (no compile); after mcb_program_jit_build (or a plan) the cached cubin is
    used — same bytes either way."""
    monkeypatch.setenv("MCB_JIT_CACHE", str(tmp_path))  # a cold disk cache
    assert gpu.program_jit(1) == 1
    p = gpu.Program("exp(-b*(x1-0.25)^2) * (1 + 0.5*sin(9*x2)) + x1", 2, ["b"])
    f = p.integrand({"b": 7.5}, n_samples=300_000, index=4)
    n0 = gpu.program_jit_compiles()
    first = gpu.run_direct([f], 17, 3)  # interpreter: not cached, too small to compile
    assert gpu.program_jit_compiles() == n0
    p.jit_build()  # all five kernel modes
    assert gpu.program_jit_compiles() == n0 + 5
    later = gpu.run_direct([f], 17, 3)  # specialised (in memory now)
    assert first.tobytes() == later.tobytes()
    q = gpu.Program("exp(-b*(x1-0.25)^2) * (1 + 0.5*sin(9*x2)) + x2", 2, ["b"])
    plan = gpu.Plan([q.integrand({"b": 7.5}, n_samples=300_000, index=4)], 17, 3)  # plans compile their mode
    assert gpu.program_jit_compiles() == n0 + 6
    plan.close()


@pytest.mark.gpu
def test_wide_random_programs_vs_reference_golden(gpu):
    """64 more random programs (dims 1-6, random boxes, up to 4 parameters,
    depth 2-5) against the reference's own values and estimates: per-sample
    values through the interpreter, estimates through both the interpreter and
    the specialised kernels."""
    with open(GOLDEN) as fh:
        cases = json.load(fh)["programs_wide"]
    keep, fns = [], []
    for c in cases:
        params, lo, hi = _case(c)
        p = gpu.Program(c["source"], c["dim"], list(params))
        keep.append(p)
        f = p.integrand(params, low=lo, high=hi, n_samples=c["n_samples"], index=c["index"])
        got = gpu.debug_eval(f, c["seed"], c["trial"], c["chunk_base"], 0, 32)
        want = np.array([fx(v) for v in c["values"]])
        assert _values_close(got, want), c["source"]
        fns.append((f, c))
    for jit in (0, 2):
        gpu.program_jit(jit)
        try:
            for f, c in fns:
                st = gpu.direct_mc(f, c["seed"], c["trial"], c["chunk_base"])
                e = c["estimate"]
                assert st.status == e["status"], (jit, c["source"])
                assert (st.n_samples, st.n_nonfinite) == (e["n_samples"], e["n_nonfinite"]), (jit, c["source"])
                if e["status"] != 0:
                    continue
                check_stats({"value": st.value, "std_error": st.std_error, "n_samples": st.n_samples,
                             "n_nonfinite": st.n_nonfinite}, fx(e["value"]), fx(e["std_error"]), e["n_samples"],
                            e["n_nonfinite"], f"programs wide (jit {jit})")
        finally:
            gpu.program_jit(1)


def test_parameter_scan_arguments(mcb):
    p = mcb.Program("a*x1 + b", 1, ["a", "b"])
    with pytest.raises(ValueError, match="not a parameter"):
        mcb.parameter_scan(p, {"a": 1.0, "b": 0.0}, "c", [1.0], 2, 1)
    with pytest.raises(ValueError, match="no values"):
        mcb.parameter_scan(p, {"a": 1.0, "b": 0.0}, "a", [], 2, 1)


@pytest.mark.gpu
def test_parameter_scan_matches_reference(gpu):
    """parameter_scan (ref src/batch.cpp:335-367) = run_batch of the expanded job: the
    reference's own run_batch on the same sources, value by value."""
    src = "cos(k*(x1+x2+x3+x4)) + sin(k*(x1+x2+x3+x4))"
    p = gpu.Program(src, 4, ["k"])
    ks = [0.5 + 0.37 * i for i in range(24)]
    out, summaries = gpu.parameter_scan(p, {}, "k", ks, 3, 77, n_samples=40_000)
    fns = [p.integrand({"k": k}, n_samples=40_000, index=i) for i, k in enumerate(ks)]
    ref, mean, _, _, _ = _oracle.ref_run_batch(fns, 77, 3, sources=[src.replace("k", repr(k)) for k in ks])
    assert np.array_equal(out["n_samples"], ref["n_samples"])
    assert np.all(np.abs(out["value"] - ref["value"]) <= 1e-12 + 1e-9 * np.abs(ref["value"]))
    assert np.allclose([s[0] for s in summaries], mean, rtol=1e-9, atol=1e-12)
    assert all(s[2] == 3 for s in summaries)


_NP_SCRIPT = r"""
import hashlib, sys
sys.path.insert(0, sys.argv[1])
import paper_2104_10073_b200 as mcb
mcb.program_jit(0)
srcs = [("cos(k*(x1+x2+x3+x4)) + sin(k*(x1+x2+x3+x4))", 4, {"k": 31.5}),
        ("exp(-3*(x1-0.4)^2) * cos(5*x2) + x3 / (x1 - 0.5)", 3, {}),
        ("pow(x1, a) * log(x2) + sqrt(x1*x2) - floor(3*x3) + min(x1, x2) * max(x2, x3) + tan(x1)", 3, {"a": 1.5}),
        ("cos(1e7*x1) + sin(1e7*x1) + sin(x2)*cos(x2) + asin(x1) + acos(x2) + atan(x1/x2)", 2, {}),
        ("((x1+x2)*(x3+x4))/((x5-x6)*(x7+x8)) + ((x1*x2)+(x3*x4))*((x5*x6)-(x7*x8))", 8, {})]
keep, fns = [], []
for i, (s, d, p) in enumerate(srcs):
    prog = mcb.Program(s, d, sorted(p))
    keep.append(prog)
    fns.append(prog.integrand(p, n_samples=150_001, index=i))
    fns.append(prog.integrand(p, low=[-0.5] * d, high=[1.5] * d, n_samples=70_000, index=10 + i))
fns.append(mcb.stratify(keep[1].integrand({}, low=[-1, 0, 0], high=[1, 2, 1], n_samples=300_000, index=30),
                        cells_per_dim=2))
# >= 1024 small cells: the lane-per-cell interpreter kernel (mode 4), odd samples per cell
fns.append(mcb.stratify(keep[0].integrand({"k": 31.5}, n_samples=1_000_000, index=31)))
fns.append(mcb.stratify(keep[1].integrand({}, n_samples=500_000, index=32), cells_per_dim=11))
# small cells of a small grid (warp per tile, mode 3) and a tree (its rounds run mode 3 too)
fns.append(mcb.stratify(keep[1].integrand({}, n_samples=200_001, index=33), cells_per_dim=5))
fns.append(mcb.tree(keep[2].integrand({"a": 1.5}, n_samples=60_000, index=34), samples_per_cell=300))
out = mcb.run_direct(fns, 4242, 3)
print(hashlib.sha256(out.tobytes()).hexdigest())
"""


@pytest.mark.gpu
def test_interpreter_pairs_per_dispatch_bit_identical(tmp_path):
    """The bytecode interpreter dispatches each instruction for NP pairs at
    once (1, 2 or 4 by the program's shared-memory need); a thread still takes
    its pairs in ascending order, so every McEstimate is byte-identical for
    any NP (forced per process with MCB_INTERP_NP; JIT off)."""
    import subprocess
    import sys
    script = tmp_path / "np.py"
    script.write_text(_NP_SCRIPT)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    digests = []
    for np_ in ("1", "2", "4"):
        env = dict(os.environ, MCB_INTERP_NP=np_, MCB_PROGRAM_JIT="0")
        r = subprocess.run([sys.executable, str(script), root], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        digests.append(r.stdout.split()[-1])
    assert digests[0] == digests[1] == digests[2], digests
