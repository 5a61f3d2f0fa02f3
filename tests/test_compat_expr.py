"""The expression front-end of the source-compatible layer (include/mcbatch/
expr.hpp, csrc/compat_mcbatch.cpp) against the reference's own
(src/expr.cpp, through oracle/_ref): the same error class for every bad
source, and for every good one the same postfix program instruction by
instruction (op, slot, constant bits), the same stack need, a bit-identical
tree_eval and an exact print -> parse round trip.  Host code only (CPU)."""
import ctypes
import os
import random
import subprocess

import pytest

from tests import _oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "_build", "test_compat_expr")

FIXED = [
    "2+3*4", "2^3^2", "2*3+4", "2^-3", "-x1^2", "-(x1)^2", "x1-x2-x3", "x1/x2/x3", "a*cos(k*(x1+x2+x3+x4)) + b*sin(k*(x1+x2+x3+x4))",
    "cos(k*(x1+x2+x3+x4)) + sin(k*(x1+x2+x3+x4))", "abs(x1+x2-x3)", "pow(x1, 2.5) + min(a, x2) - max(b, 1e-3)",
    "exp(-100*((x1-0.5)^2+(x2-0.5)^2))", "sqrt(abs(x1)) * floor(x2 * 10) / 10", "pi * e", "1.5e3 + 2E-2 + 3.",
    "asin(x1/3) + acos(x2/3) + atan(x3) + tan(x1) + log(2 + x2)", "x10", "--x1", "x1 ^ -x2 ^ 2", "1e", "2ee",
    # errors
    "", "   ", "x1 +", "(x1", "x1)", "foo(x1)", "sin x1", "sin(x1, x2)", "pow(x1)", "x0 + 1", "x1 $ 2",
    "x4", "q + x1", "min()", "3 4", "x1 @", ",", "x01",
]


def _rand_expr(rng, depth=0, dim=3, params=("a", "b")):
    roll = rng.randrange(100)
    if depth >= 4 or roll < 35:
        k = rng.randrange(3)
        if k == 0:
            return repr(round(rng.uniform(0, 4), rng.randrange(1, 17)))
        if k == 1:
            return f"x{rng.randrange(1, dim + 1)}"
        return rng.choice(params)
    if roll < 45:
        return "-" + _rand_expr(rng, depth + 1, dim, params)
    if roll < 75:
        op = rng.choice("+-*/^")
        return f"({_rand_expr(rng, depth + 1, dim, params)} {op} {_rand_expr(rng, depth + 1, dim, params)})"
    fn = rng.choice(["sin", "cos", "tan", "atan", "exp", "log", "sqrt", "abs", "floor", "asin", "acos",
                     "pow", "min", "max"])
    if fn in ("pow", "min", "max"):
        return f"{fn}({_rand_expr(rng, depth + 1, dim, params)}, {_rand_expr(rng, depth + 1, dim, params)})"
    return f"{fn}({_rand_expr(rng, depth + 1, dim, params)})"


def _build():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    lib = os.path.join(ROOT, "paper_2104_10073_b200")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_compat_expr.cpp"), "-L" + lib, "-l:libmcb.so",
                    "-Wl,-rpath," + lib, "-o", EXE], check=True)


def _cases():
    rng = random.Random(20261018)
    cases = []
    for src in FIXED:
        cases.append((3, ["a", "b", "k"], src))
    for _ in range(400):
        cases.append((3, ["a", "b"], _rand_expr(rng)))
    out = []
    for dim, names, src in cases:
        point = [rng.uniform(-2, 2) for _ in range(dim)]
        params = [rng.uniform(-2, 2) for _ in names]
        out.append((dim, names, src, point, params))
    return out


@pytest.mark.skipif(_oracle.load_ref() is None, reason="reference library not built")
def test_expr_front_end_matches_reference():
    _build()
    ref = _oracle.load_ref()
    ref.ref_expr_dump.restype = ctypes.c_int
    ref.ref_expr_dump.argtypes = [ctypes.c_char_p, ctypes.c_uint32, ctypes.c_char_p, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t]
    cases = _cases()
    lines = []
    want = []
    for dim, names, src, point, params in cases:
        lines.append(f"{dim}|{','.join(names)}|{src}|{';'.join(repr(p) for p in point)}|"
                     f"{';'.join(repr(p) for p in params)}")
        pt = (ctypes.c_double * dim)(*point)
        pv = (ctypes.c_double * max(1, len(params)))(*params)
        buf = ctypes.create_string_buffer(1 << 16)
        ref.ref_expr_dump(src.encode(), dim, ",".join(names).encode(), pt, pv, buf, len(buf))
        want.append(buf.value.decode())
    r = subprocess.run([EXE], input="\n".join(lines) + "\n", capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    got = r.stdout.splitlines()
    assert len(got) == len(want)
    n_ok = 0
    for (dim, names, src, _, _), g, w in zip(cases, got, want):
        assert g == w, (src, g, w)
        n_ok += g.startswith("OK")
    assert n_ok > 350  # most random programs compile; every error class above is exercised
