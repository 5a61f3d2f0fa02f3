"""Pure-Python restatement of the reference DSL (TEST INFRASTRUCTURE ONLY).

Restates ref/src/expr.cpp: the lexer/recursive-descent parser (:108-300),
postfix compilation (:442-518) and the postfix interpreter
`CompiledProgram::evaluate` (:520-553) with glibc math through Python's
`math` module, plus Welford accumulation (ref/src/estimator.cpp:9-49) for
small direct-MC estimates.  Pinned bit-exactly against values produced by the
reference itself (tests/golden/golden.json "programs").  Small cases only
(pure-Python loops); used as the checker of the GPU interpreter.
"""
from __future__ import annotations

import math

FUNCS = {"sin": 1, "cos": 1, "tan": 1, "asin": 1, "acos": 1, "atan": 1, "exp": 1, "log": 1,
         "sqrt": 1, "abs": 1, "floor": 1, "pow": 2, "min": 2, "max": 2}


class DslError(Exception):
    pass


def _lex(src):
    toks, i = [], 0
    while True:
        while i < len(src) and src[i].isspace():
            i += 1
        if i >= len(src):
            toks.append(("end", None, i))
            return toks
        c = src[i]
        if c in "+-*/^(),":
            toks.append((c, None, i))
            i += 1
        elif c.isdigit():
            j = i
            while j < len(src) and src[j].isdigit():
                j += 1
            if j < len(src) and src[j] == ".":
                j += 1
                while j < len(src) and src[j].isdigit():
                    j += 1
            if j < len(src) and src[j] in "eE":
                k = j + 1
                if k < len(src) and src[k] in "+-":
                    k += 1
                if k < len(src) and src[k].isdigit():
                    j = k
                    while j < len(src) and src[j].isdigit():
                        j += 1
            toks.append(("num", float(src[i:j]), i))
            i = j
        elif c.isalpha() or c == "_":
            j = i
            while j < len(src) and (src[j].isalnum() or src[j] == "_"):
                j += 1
            toks.append(("id", src[i:j], i))
            i = j
        else:
            raise DslError(f"unexpected character '{c}'")


def parse(src):
    """AST as nested tuples: ('num', v) ('var', j) ('par', name) ('neg', e)
    ('bin', op, l, r) ('call', name, [args])."""
    if not src:
        raise DslError("empty expression")
    toks = _lex(src)
    pos = [0]

    def peek():
        return toks[pos[0]][0]

    def take():
        t = toks[pos[0]]
        pos[0] += 1
        return t

    def expr():
        l = term()
        while peek() in "+-" and peek() != "end":
            op = take()[0]
            l = ("bin", op, l, term())
        return l

    def term():
        l = factor()
        while peek() in ("*", "/"):
            op = take()[0]
            l = ("bin", op, l, factor())
        return l

    def factor():
        b = unary()
        if peek() == "^":
            take()
            return ("bin", "^", b, factor())
        return b

    def unary():
        if peek() == "-":
            take()
            return ("neg", unary())
        return primary()

    def primary():
        kind, val, _ = take()
        if kind == "num":
            return ("num", val)
        if kind == "(":
            e = expr()
            if take()[0] != ")":
                raise DslError("expected ')'")
            return e
        if kind != "id":
            raise DslError("expected a number, identifier or '('")
        name = val
        if peek() == "(":
            if name not in FUNCS:
                raise DslError(f"unknown function '{name}'")
            take()
            args = [expr()]
            while peek() == ",":
                take()
                args.append(expr())
            if take()[0] != ")":
                raise DslError("expected ')'")
            if len(args) != FUNCS[name]:
                raise DslError(f"function '{name}' expects {FUNCS[name]} argument(s)")
            return ("call", name, args)
        if name in FUNCS:
            raise DslError(f"expected '(' after function name '{name}'")
        if name == "pi":
            return ("num", math.pi)
        if name == "e":
            return ("num", math.e)
        if len(name) >= 2 and name[0] == "x" and name[1] in "123456789" and name[1:].isdigit():
            return ("var", int(name[1:]) - 1)
        return ("par", name)

    e = expr()
    if peek() != "end":
        raise DslError("unexpected trailing input")
    return e


def compile_postfix(ast, dim, param_names):
    """Postfix list [(op, arg)] in the reference's emission order."""
    names = sorted(param_names)
    code = []

    def emit(n):
        k = n[0]
        if k == "num":
            code.append(("const", n[1]))
        elif k == "var":
            if n[1] >= dim:
                raise DslError(f"x{n[1] + 1} exceeds dim={dim}")
            code.append(("var", n[1]))
        elif k == "par":
            if n[1] not in names:
                raise DslError(f"unbound parameter '{n[1]}'")
            code.append(("par", names.index(n[1])))
        elif k == "neg":
            emit(n[1])
            code.append(("neg", None))
        elif k == "bin":
            emit(n[2])
            emit(n[3])
            code.append((n[1], None))
        else:
            for a in n[2]:
                emit(a)
            code.append((n[1], None))

    emit(ast)
    return code


_UN = {"neg": lambda a: -a, "sin": math.sin, "cos": math.cos, "tan": math.tan, "asin": math.asin,
       "acos": math.acos, "atan": math.atan, "exp": math.exp, "log": math.log, "sqrt": math.sqrt,
       "abs": math.fabs, "floor": math.floor}


def _odd_integer(b):
    return math.isfinite(b) and float(b).is_integer() and int(b) % 2 == 1


def _pow(a, b):
    """C99/glibc pow where Python's math.pow raises."""
    try:
        return math.pow(a, b)
    except ValueError:
        if a == 0 and b < 0:  # pole: +-inf, sign kept for odd integer exponents
            return math.copysign(math.inf, a) if _odd_integer(b) else math.inf
        return math.nan  # negative base, non-integer exponent
    except OverflowError:
        return -math.inf if (a < 0 and _odd_integer(b)) else math.inf


def _safe_un(f, a):
    if f is math.floor and not math.isfinite(a):
        return a
    try:
        return float(f(a))
    except ValueError:
        if f is math.log and a == 0:
            return -math.inf
        return math.nan
    except OverflowError:
        return math.inf


def _fmin(a, b):
    if math.isnan(a):
        return b
    if math.isnan(b):
        return a
    return min(a, b)


def _fmax(a, b):
    if math.isnan(a):
        return b
    if math.isnan(b):
        return a
    return max(a, b)


_BIN = {"+": lambda a, b: a + b, "-": lambda a, b: a - b, "*": lambda a, b: a * b,
        "/": lambda a, b: (a / b) if b != 0 else (math.copysign(math.inf, a) * math.copysign(1.0, b)
                                                  if a != 0 and not math.isnan(a) else math.nan),
        "^": _pow, "pow": _pow, "min": _fmin, "max": _fmax}


def evaluate(code, x, params):
    """CompiledProgram::evaluate (ref/src/expr.cpp:520-553), scalar, glibc math."""
    st = []
    for op, arg in code:
        if op == "const":
            st.append(arg)
        elif op == "var":
            st.append(x[arg])
        elif op == "par":
            st.append(params[arg])
        elif op in _UN:
            st.append(_safe_un(_UN[op], st.pop()))
        else:
            b = st.pop()
            a = st.pop()
            try:
                st.append(float(_BIN[op](a, b)))
            except OverflowError:
                st.append(math.inf)
    return st[0]


class Program:
    def __init__(self, source, dim, params: dict):
        self.source, self.dim = source, dim
        self.names = sorted(params)
        self.values = [params[n] for n in self.names]
        self.code = compile_postfix(parse(source), dim, self.names)

    def __call__(self, x):
        return evaluate(self.code, x, self.values)


def welford_direct_mc(values_by_chunk, volume):
    """accumulate_chunk + reduce_chunks (ref/src/estimator.cpp:9-73) over
    per-chunk value lists; returns (value, std_error, n_samples, n_nonfinite)."""
    n_tot, nn_tot, mean_tot, m2_tot = 0, 0, 0.0, 0.0
    for vals in values_by_chunk:
        n, nn, mean, m2 = 0, 0, 0.0, 0.0
        for v in vals:
            if not math.isfinite(v):
                nn += 1
                continue
            n += 1
            d = v - mean
            mean += d / n
            m2 += d * (v - mean)
        nn_tot += nn
        if n == 0:
            continue
        if n_tot == 0:
            n_tot, mean_tot, m2_tot = n, mean, m2
            continue
        d = mean - mean_tot
        tot = n_tot + n
        mean_tot += d * (n / tot)
        m2_tot += m2 + d * d * (n_tot * n / tot)
        n_tot = tot
    if n_tot == 0:
        return None
    se = volume * math.sqrt((m2_tot / (n_tot - 1)) / n_tot) if n_tot >= 2 else math.inf
    return volume * mean_tot, se, n_tot + nn_tot, nn_tot
