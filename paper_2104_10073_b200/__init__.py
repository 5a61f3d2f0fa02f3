"""B200-native direct Monte Carlo multi-function integration (arXiv 2104.10073).

Python view of the C-ABI in ``include/mcb/mcb.h`` (ctypes over the in-tree
``libmcb.so``).  The library is the product: sm_100a kernels behind a C ABI,
with no CPU fallback — importing this package without the built library
raises, and compute calls without a B200 return ``MCB_ERR_NO_DEVICE``.

Reference correspondence (``/root/reference/proj``):
``run_direct`` ~ ``run_batch`` Direct branch (src/batch.cpp:195-333),
``direct_mc`` ~ src/estimator.cpp:75-92, ``tree_refine`` ~ src/estimator.cpp:212-318,
``debug_points`` ~ ``sample_uniform``
(src/sampling.cpp:102-112), ``make_harmonic_job`` ~ src/job_io.cpp:355-376.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MCB_LIB") or os.path.join(_HERE, "libmcb.so")

CHUNK_SIZE = 65536
MAX_DIM = 8

FAMILY_HARMONIC = 0
FAMILY_HARMONIC_VEC = 1
FAMILY_ABS2 = 2
FAMILY_ABS3 = 3
FAMILY_PROGRAM = 4
FLAG_UNIT_COEFFS = 1
FLAG_REFINE_CONFIG = 2
MAX_PARAMS = 8

TRIAL_OK = 0
TRIAL_ALL_NONFINITE = 1
TRIAL_DEAD_CELL = 2
TRIAL_CELL_BUDGET = 3
TRIAL_CHUNK_RANGE = 4

METHOD_DIRECT = 0
METHOD_STRATIFIED = 1
METHOD_TREE = 2

STATUS = {0: "MCB_OK", 1: "MCB_ERR_INVALID_ARGUMENT", 2: "MCB_ERR_VALIDATION", 3: "MCB_ERR_CUDA",
          4: "MCB_ERR_NO_DEVICE", 5: "MCB_ERR_OUT_OF_RANGE", 6: "MCB_ERR_BUFFER_TOO_SMALL"}


class McbError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status


class Integrand(ctypes.Structure):
    """``mcb_integrand`` (include/mcb/mcb.h)."""
    _fields_ = [("family", ctypes.c_uint32), ("dim", ctypes.c_uint32),
                ("integrand_index", ctypes.c_uint32), ("flags", ctypes.c_uint32),
                ("n_samples", ctypes.c_uint64), ("a", ctypes.c_double), ("b", ctypes.c_double),
                ("k", ctypes.c_double * MAX_DIM), ("low", ctypes.c_double * MAX_DIM),
                ("high", ctypes.c_double * MAX_DIM), ("program", ctypes.c_void_p),
                ("method", ctypes.c_uint32), ("cells_per_dim", ctypes.c_uint32),
                ("cell_cap", ctypes.c_uint64), ("samples_per_cell", ctypes.c_uint32),
                ("max_depth", ctypes.c_uint32), ("sigma_multiplier", ctypes.c_double)]


class TrialStats(ctypes.Structure):
    """``mcb_trial_stats`` = reference McEstimate + status."""
    _fields_ = [("value", ctypes.c_double), ("std_error", ctypes.c_double),
                ("n_samples", ctypes.c_uint64), ("n_nonfinite", ctypes.c_uint64),
                ("status", ctypes.c_uint32), ("nonfinite_warning", ctypes.c_uint32),
                ("detail", ctypes.c_uint32), ("n_cells", ctypes.c_uint32),
                ("budget_exhausted", ctypes.c_uint32), ("max_depth", ctypes.c_uint32)]


class ChunkAccum(ctypes.Structure):
    """``mcb_chunk_accum`` = reference ChunkAccum (include/mcbatch/estimator.hpp:60-68)."""
    _fields_ = [("n", ctypes.c_uint64), ("n_nonfinite", ctypes.c_uint64),
                ("mean", ctypes.c_double), ("m2", ctypes.c_double)]


class Leaf(ctypes.Structure):
    """``mcb_leaf`` = reference StratumNode (include/mcbatch/estimator.hpp:33-38)."""
    _fields_ = [("low", ctypes.c_double * MAX_DIM), ("high", ctypes.c_double * MAX_DIM),
                ("estimate", TrialStats), ("depth", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


class Violation(ctypes.Structure):
    _fields_ = [("integrand", ctypes.c_int64), ("message", ctypes.c_char * 120)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("n_fns", ctypes.c_uint64), ("trials", ctypes.c_uint32),
                ("n_groups", ctypes.c_uint32), ("n_tiles", ctypes.c_uint64),
                ("total_samples", ctypes.c_uint64), ("philox_blocks", ctypes.c_uint64),
                ("launches_per_run", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


TRIAL_DTYPE = np.dtype([("value", "<f8"), ("std_error", "<f8"), ("n_samples", "<u8"),
                        ("n_nonfinite", "<u8"), ("status", "<u4"), ("nonfinite_warning", "<u4"),
                        ("detail", "<u4"), ("n_cells", "<u4"), ("budget_exhausted", "<u4"),
                        ("max_depth", "<u4")])
assert TRIAL_DTYPE.itemsize == ctypes.sizeof(TrialStats)

# Every symbol include/mcb/mcb.h declares (checked by tests/test_abi.py).
ABI_SYMBOLS = [
    "mcb_abi_version", "mcb_last_error", "mcb_device_count", "mcb_stream_key", "mcb_volume",
    "mcb_to_dsl", "mcb_validate", "mcb_partition", "mcb_summarize_trials", "mcb_run_direct",
    "mcb_direct_mc", "mcb_plan_create", "mcb_plan_launch", "mcb_plan_download",
    "mcb_plan_get_info", "mcb_plan_destroy", "mcb_debug_points", "mcb_debug_eval",
    "mcb_probe_philox_peak", "mcb_program_compile", "mcb_program_destroy", "mcb_program_info",
    "mcb_program_param_name", "mcb_stratified_plan", "mcb_tree_refine", "mcb_program_jit",
    "mcb_program_jit_compiles", "mcb_program_jit_error", "mcb_program_jit_build", "mcb_stratified_mc",
    "mcb_program_eval_points", "mcb_accumulate_chunk",
]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(or make -C paper_2104_10073_b200/csrc). There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    u32, u64, i32, dbl, vp, sz = (ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_double,
                                  ctypes.c_void_p, ctypes.c_size_t)
    sig = {
        "mcb_abi_version": (u32, []),
        "mcb_last_error": (ctypes.c_char_p, []),
        "mcb_device_count": (i32, []),
        "mcb_stream_key": (None, [u64, u32, P(u32)]),
        "mcb_volume": (dbl, [P(Integrand)]),
        "mcb_to_dsl": (sz, [P(Integrand), ctypes.c_char_p, sz]),
        "mcb_validate": (i32, [P(Integrand), sz, P(ctypes.c_char_p), u32, P(Violation), sz, P(sz)]),
        "mcb_partition": (i32, [P(Integrand), sz, u32, i32, P(u32)]),
        "mcb_summarize_trials": (i32, [P(TrialStats), u32, P(dbl), P(dbl), P(u32)]),
        "mcb_run_direct": (i32, [P(Integrand), sz, u64, u32, P(i32), i32, vp, P(dbl)]),
        "mcb_direct_mc": (i32, [P(Integrand), u64, u32, u64, i32, P(TrialStats)]),
        "mcb_accumulate_chunk": (i32, [P(Integrand), u64, u32, u64, u32, i32, P(ChunkAccum)]),
        "mcb_plan_create": (i32, [P(Integrand), sz, u64, u32, i32, P(vp)]),
        "mcb_plan_launch": (i32, [vp, vp]),
        "mcb_plan_download": (i32, [vp, vp, vp]),
        "mcb_plan_get_info": (i32, [vp, P(PlanInfo)]),
        "mcb_plan_destroy": (None, [vp]),
        "mcb_debug_points": (i32, [u64, u32, u32, u64, u64, u64, u32, P(dbl), P(dbl), i32, vp]),
        "mcb_debug_eval": (i32, [P(Integrand), u64, u32, u64, u64, u64, i32, vp]),
        "mcb_probe_philox_peak": (i32, [i32, dbl, P(dbl)]),
        "mcb_program_compile": (i32, [ctypes.c_char_p, u32, P(ctypes.c_char_p), sz, P(vp)]),
        "mcb_program_destroy": (None, [vp]),
        "mcb_program_eval_points": (i32, [vp, P(ctypes.c_double), sz, vp, u64, i32, vp]),
        "mcb_program_info": (i32, [vp, P(u32), P(u32), P(u32)]),
        "mcb_program_param_name": (sz, [vp, u32, ctypes.c_char_p, sz]),
        "mcb_stratified_plan": (i32, [P(Integrand), P(u32), P(u64), P(u32)]),
        "mcb_tree_refine": (i32, [P(Integrand), u64, u32, u64, i32, P(TrialStats), P(Leaf), sz, P(sz)]),
        "mcb_program_jit": (i32, [i32]),
        "mcb_program_jit_compiles": (u64, []),
        "mcb_program_jit_error": (sz, [ctypes.c_char_p, sz]),
        "mcb_program_jit_build": (i32, [vp]),
        "mcb_stratified_mc": (i32, [P(Integrand), u32, u32, u64, u64, u32, u64, i32, P(TrialStats), P(Leaf), sz,
                                    P(sz)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def _check(status: int) -> None:
    if status != 0:
        raise McbError(status, lib.mcb_last_error().decode())


def device_count() -> int:
    return int(lib.mcb_device_count())


# ---------------------------------------------------------------- descriptors

def make_integrand(family: int, dim: int, *, k=0.0, a: float = 1.0, b: float = 1.0,
                   low: Optional[Sequence[float]] = None, high: Optional[Sequence[float]] = None,
                   n_samples: int = 10000, index: int = 0, unit_coeffs: bool = False) -> Integrand:
    f = Integrand()
    f.family, f.dim, f.integrand_index = family, dim, index
    f.flags = FLAG_UNIT_COEFFS if unit_coeffs else 0
    f.n_samples = n_samples
    f.a, f.b = a, b
    ks = list(k) if isinstance(k, (list, tuple, np.ndarray)) else [k]
    for j, v in enumerate(ks):
        f.k[j] = v
    lo = [0.0] * dim if low is None else list(low)
    hi = [1.0] * dim if high is None else list(high)
    for j in range(dim):
        f.low[j], f.high[j] = lo[j], hi[j]
    return f


def harmonic(k: float, dim: int = 4, *, a: float = 1.0, b: float = 1.0, unit_coeffs=None,
             low=None, high=None, n_samples: int = 10000, index: int = 0) -> Integrand:
    """a*cos(k*(x1+..+xd)) + b*sin(k*(x1+..+xd)); unit_coeffs -> the Fig.1 form."""
    if unit_coeffs is None:
        unit_coeffs = (a == 1.0 and b == 1.0)
    return make_integrand(FAMILY_HARMONIC, dim, k=k, a=a, b=b, low=low, high=high,
                          n_samples=n_samples, index=index, unit_coeffs=unit_coeffs)


class Program:
    """A compiled DSL integrand (``mcb_program_compile``): the reference's
    source language (ref/src/expr.cpp), run on the GPU by the interpreter
    kernel.  Parameters bind in sorted-name order; keep the object alive while
    integrands reference it."""

    def __init__(self, source: str, dim: int, param_names: Sequence[str] = ()):
        names = sorted(set(param_names))
        arr = (ctypes.c_char_p * max(1, len(names)))(*[n.encode() for n in names])
        h = ctypes.c_void_p()
        _check(lib.mcb_program_compile(source.encode(), dim, arr, len(names), ctypes.byref(h)))
        self._h = h
        self.source, self.dim = source, dim
        n_instr, depth, n_params = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
        _check(lib.mcb_program_info(h, ctypes.byref(n_instr), ctypes.byref(depth), ctypes.byref(n_params)))
        self.n_instr, self.depth = n_instr.value, depth.value
        self.param_names = []
        for i in range(n_params.value):
            buf = ctypes.create_string_buffer(lib.mcb_program_param_name(h, i, None, 0))
            lib.mcb_program_param_name(h, i, buf, len(buf))
            self.param_names.append(buf.value.decode())

    @property
    def handle(self) -> int:
        return self._h.value

    def integrand(self, params: Optional[Dict[str, float]] = None, *, low=None, high=None,
                  n_samples: int = 10000, index: int = 0) -> Integrand:
        params = params or {}
        missing = [n for n in self.param_names if n not in params]
        if missing:
            raise ValueError(f"unbound parameter '{missing[0]}'")
        f = make_integrand(FAMILY_PROGRAM, self.dim, k=[params[n] for n in self.param_names] or 0.0,
                           low=low, high=high, n_samples=n_samples, index=index)
        f.program = self._h.value
        f.a = f.b = 0.0
        f._program_ref = self  # the descriptor holds the raw handle: keep the program alive
        return f

    def evaluate(self, points, params: Optional[Dict[str, float]] = None, device: int = 0) -> np.ndarray:
        """CompiledProgram::evaluate (ref src/expr.cpp:520-553) at the given
        points ((n, dim) array) on the GPU interpreter the estimators use."""
        params = params or {}
        missing = [n for n in self.param_names if n not in params]
        if missing:
            raise ValueError(f"unbound parameter '{missing[0]}'")
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, self.dim)
        pv = (ctypes.c_double * max(1, len(self.param_names)))(*[params[n] for n in self.param_names])
        out = np.zeros(len(pts))
        _check(lib.mcb_program_eval_points(self._h, pv, len(self.param_names), pts.ctypes.data, len(pts), device,
                                           out.ctypes.data))
        return out

    def jit_build(self) -> None:
        """NVRTC-compile this program's specialised kernels now (no device needed)."""
        _check(lib.mcb_program_jit_build(self._h))

    def close(self):
        if getattr(self, "_h", None):
            lib.mcb_program_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def to_dsl(f: Integrand) -> str:
    n = lib.mcb_to_dsl(ctypes.byref(f), None, 0)
    buf = ctypes.create_string_buffer(n)
    lib.mcb_to_dsl(ctypes.byref(f), buf, n)
    return buf.value.decode()


def volume(f: Integrand) -> float:
    return float(lib.mcb_volume(ctypes.byref(f)))


def stream_key(seed: int, integrand_index: int):
    key = (ctypes.c_uint32 * 2)()
    lib.mcb_stream_key(seed, integrand_index, key)
    return int(key[0]), int(key[1])


def as_array(fns: Sequence[Integrand]):
    if isinstance(fns, ctypes.Array):
        return fns
    arr = (Integrand * len(fns))()
    for i, f in enumerate(fns):
        arr[i] = f
    # programs referenced by raw handle stay alive as long as the array
    arr._programs = [p for p in {id(p): p for p in (getattr(f, "_program_ref", None) for f in fns)}.values()
                     if p is not None]
    return arr


def validate(fns: Sequence[Integrand], trials: int, names: Optional[Sequence[str]] = None):
    arr = as_array(fns)
    cap = 8 * len(arr) + 8
    out = (Violation * cap)()
    n = ctypes.c_size_t()
    cn = None
    if names is not None:
        cn = (ctypes.c_char_p * len(names))(*[s.encode() for s in names])
    _check(lib.mcb_validate(arr, len(arr), cn, trials, out, cap, ctypes.byref(n)))
    return [(int(out[i].integrand), out[i].message.decode()) for i in range(min(n.value, cap))]


def stratify(f: Integrand, cells_per_dim: int = 0, cell_cap: int = 0) -> Integrand:
    """Switch an integrand to the stratified method (ref src/estimator.cpp:161-182)."""
    f.method = METHOD_STRATIFIED
    f.cells_per_dim = cells_per_dim
    f.cell_cap = cell_cap
    return f


def tree(f: Integrand, *, init_cells_per_dim: int = 0, samples_per_cell: int = 2048,
         max_depth: int = 6, sigma_multiplier: float = 1.0, cell_cap: int = 0) -> Integrand:
    """Switch an integrand to the adaptive tree method (ref src/estimator.cpp:212-318);
    its n_samples is the refinement budget.  Defaults = RefineConfig's."""
    f.method = METHOD_TREE
    f.cells_per_dim = init_cells_per_dim
    f.cell_cap = cell_cap
    f.flags |= FLAG_REFINE_CONFIG
    f.samples_per_cell = samples_per_cell
    f.max_depth = max_depth
    f.sigma_multiplier = sigma_multiplier
    return f


def stratified_plan(f: Integrand):
    """(cells_per_dim, n_cells, samples_per_cell) — ref src/batch.cpp:41-54."""
    k, n, spc = ctypes.c_uint32(), ctypes.c_uint64(), ctypes.c_uint32()
    _check(lib.mcb_stratified_plan(ctypes.byref(f), ctypes.byref(k), ctypes.byref(n), ctypes.byref(spc)))
    return k.value, n.value, spc.value


def partition(fns: Sequence[Integrand], trials: int, n_shards: int) -> np.ndarray:
    arr = as_array(fns)
    out = (ctypes.c_uint32 * len(arr))()
    _check(lib.mcb_partition(arr, len(arr), trials, n_shards, out))
    return np.frombuffer(out, dtype=np.uint32).copy()


def summarize_trials(per_trial: np.ndarray):
    arr = np.ascontiguousarray(per_trial, dtype=TRIAL_DTYPE)
    mean, sd, nok = ctypes.c_double(), ctypes.c_double(), ctypes.c_uint32()
    _check(lib.mcb_summarize_trials(arr.ctypes.data_as(ctypes.POINTER(TrialStats)), len(arr),
                                    ctypes.byref(mean), ctypes.byref(sd), ctypes.byref(nok)))
    return mean.value, sd.value, nok.value


# ---------------------------------------------------------------- hot path

def run_direct(fns: Sequence[Integrand], seed: int, trials: int,
               devices: Optional[Sequence[int]] = None, return_seconds: bool = False):
    """All integrands x trials on the GPU(s); returns a (n_fns, trials) TRIAL_DTYPE array."""
    arr = as_array(fns)
    out = np.zeros((len(arr), trials), dtype=TRIAL_DTYPE)
    secs = ctypes.c_double()
    if devices:
        dv = (ctypes.c_int * len(devices))(*devices)
        nd = len(devices)
    else:
        dv, nd = None, 0
    _check(lib.mcb_run_direct(arr, len(arr), seed, trials, dv, nd, out.ctypes.data,
                              ctypes.byref(secs)))
    return (out, secs.value) if return_seconds else out


def parameter_scan(program: "Program", params: Dict[str, float], name: str, values: Sequence[float],
                   trials: int, seed: int, *, low=None, high=None, n_samples: int = 10000,
                   devices: Optional[Sequence[int]] = None):
    """parameter_scan (ref include/mcbatch/batch.hpp:76-81, src/batch.cpp:335-367): the
    template program once per value of parameter `name` (integrand_index = the value's
    position, as in the reference's `name#i` job), run as one batch.  Returns the
    (len(values), trials) per-trial array and one (mean, trial_stddev, n_ok) per value."""
    if name not in program.param_names:
        raise ValueError(f"parameter '{name}' is not a parameter of the template")
    if len(values) == 0:
        raise ValueError("no values to scan")
    fns = [program.integrand({**params, name: float(v)}, low=low, high=high, n_samples=n_samples, index=i)
           for i, v in enumerate(values)]
    out = run_direct(fns, seed, trials, devices)
    # the reference's success rule (src/batch.cpp:320-329): with two or more
    # trials an integrand needs at least two successful ones, else one; a
    # failed integrand makes the scan throw (src/batch.cpp:360-364)
    need = 2 if trials >= 2 else 1
    summaries = []
    for i, row in enumerate(out):
        n_ok = int((row["status"] == TRIAL_OK).sum())
        if n_ok < need:
            bad = [f"trial {t}: status {int(row[t]['status'])}" for t in range(trials) if row[t]["status"] != TRIAL_OK]
            raise RuntimeError(f"parameter_scan: {name}#{i} failed: {n_ok} of {trials} trials succeeded "
                               f"({'; '.join(bad)})")
        summaries.append(summarize_trials(row))
    return out, summaries


def direct_mc(f: Integrand, seed: int, trial: int = 0, chunk_base: int = 0, device: int = 0):
    st = TrialStats()
    _check(lib.mcb_direct_mc(ctypes.byref(f), seed, trial, chunk_base, device, ctypes.byref(st)))
    return st


def accumulate_chunk(f: Integrand, seed: int, trial: int, chunk: int, count: int,
                     device: int = 0) -> ChunkAccum:
    """accumulate_chunk (ref src/estimator.cpp:36-49): one chunk's (n, n_nonfinite,
    mean, m2) of the stream {seed, f.integrand_index, trial, chunk}, on the GPU."""
    acc = ChunkAccum()
    _check(lib.mcb_accumulate_chunk(ctypes.byref(f), seed, trial, chunk, count, device, ctypes.byref(acc)))
    return acc


def tree_refine(f: Integrand, seed: int, trial: int = 0, chunk_base: int = 0, device: int = 0,
                leaves: bool = False):
    """tree_refine (ref src/estimator.cpp:212-318) of one integrand on the GPU.
    Returns the TrialStats, or (TrialStats, [Leaf]) with ``leaves=True``."""
    st = TrialStats()
    n = ctypes.c_size_t()
    if not leaves:
        _check(lib.mcb_tree_refine(ctypes.byref(f), seed, trial, chunk_base, device, ctypes.byref(st), None, 0,
                                   ctypes.byref(n)))
        return st
    # one call when the leaves fit the bound (first pass <= 4096 cells or the
    # given grid, plus one leaf per affordable split); the tree runs again only
    # if they do not
    spc = max(2, f.samples_per_cell if f.flags & FLAG_REFINE_CONFIG else 2048)
    grid = f.cells_per_dim ** f.dim if f.cells_per_dim else 4096
    cap = int(min(1 << 22, grid + f.n_samples // spc + 1))
    buf = (Leaf * cap)()
    _check(lib.mcb_tree_refine(ctypes.byref(f), seed, trial, chunk_base, device, ctypes.byref(st), buf, cap,
                               ctypes.byref(n)))
    if n.value > cap:
        buf = (Leaf * n.value)()
        _check(lib.mcb_tree_refine(ctypes.byref(f), seed, trial, chunk_base, device, ctypes.byref(st), buf,
                                   n.value, ctypes.byref(n)))
    return st, list(buf[:n.value])


def stratified_mc(f: Integrand, cells_per_dim: int, samples_per_cell: int, seed: int, trial: int = 0,
                  chunk_base: int = 0, cell_cap: int = 0, device: int = 0):
    """stratified_mc (ref src/estimator.cpp:161-182) on the GPU: (TrialStats, [Leaf])."""
    st = TrialStats()
    n = ctypes.c_size_t()
    cap = int(min(1 << 22, max(1, cells_per_dim) ** f.dim))
    buf = (Leaf * cap)()
    _check(lib.mcb_stratified_mc(ctypes.byref(f), cells_per_dim, samples_per_cell, cell_cap, seed, trial,
                                 chunk_base, device, ctypes.byref(st), buf, cap, ctypes.byref(n)))
    if n.value > cap:
        buf = (Leaf * n.value)()
        _check(lib.mcb_stratified_mc(ctypes.byref(f), cells_per_dim, samples_per_cell, cell_cap, seed, trial,
                                     chunk_base, device, ctypes.byref(st), buf, n.value, ctypes.byref(n)))
    return st, list(buf[:n.value])


class Plan:
    """Device-resident plan: descriptors and tile tables stay in HBM; ``launch``
    enqueues the fused kernels on a CUDA stream (a ``torch.cuda.Stream``'s
    ``cuda_stream`` handle or 0 for the legacy default stream)."""

    def __init__(self, fns: Sequence[Integrand], seed: int, trials: int, device: int = 0):
        self._arr = as_array(fns)
        self.trials = trials
        h = ctypes.c_void_p()
        _check(lib.mcb_plan_create(self._arr, len(self._arr), seed, trials, device, ctypes.byref(h)))
        self._h = h

    def info(self) -> PlanInfo:
        i = PlanInfo()
        _check(lib.mcb_plan_get_info(self._h, ctypes.byref(i)))
        return i

    def launch(self, stream: int = 0) -> None:
        _check(lib.mcb_plan_launch(self._h, ctypes.c_void_p(stream)))

    def download(self, stream: int = 0) -> np.ndarray:
        out = np.zeros((len(self._arr), self.trials), dtype=TRIAL_DTYPE)
        _check(lib.mcb_plan_download(self._h, out.ctypes.data, ctypes.c_void_p(stream)))
        return out

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.mcb_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def debug_points(seed: int, integrand_index: int, trial: int, chunk: int, first_point: int,
                 count: int, low: Sequence[float], high: Sequence[float], device: int = 0):
    dim = len(low)
    out = np.zeros((count, dim), dtype=np.float64)
    lo = (ctypes.c_double * dim)(*low)
    hi = (ctypes.c_double * dim)(*high)
    _check(lib.mcb_debug_points(seed, integrand_index, trial, chunk, first_point, count, dim, lo, hi,
                                device, out.ctypes.data))
    return out


def debug_eval(f: Integrand, seed: int, trial: int, chunk: int, first_point: int, count: int,
               device: int = 0):
    out = np.zeros(count, dtype=np.float64)
    _check(lib.mcb_debug_eval(ctypes.byref(f), seed, trial, chunk, first_point, count, device,
                              out.ctypes.data))
    return out


def program_jit(mode: int = -1) -> int:
    """Runtime specialisation of DSL programs (NVRTC): 0 off (bytecode
    interpreter), 1 automatic (default: cached / plan / large launches),
    2 always, -1 query.  Returns the active mode (0 without NVRTC)."""
    return int(lib.mcb_program_jit(mode))


def program_jit_compiles() -> int:
    return int(lib.mcb_program_jit_compiles())


def program_jit_error() -> str:
    buf = ctypes.create_string_buffer(lib.mcb_program_jit_error(None, 0))
    lib.mcb_program_jit_error(buf, len(buf))
    return buf.value.decode()


def probe_philox_peak(device: int = 0, ms: float = 50.0) -> float:
    """Philox4x32-10 blocks/s the device generates with no integrand work."""
    v = ctypes.c_double()
    _check(lib.mcb_probe_philox_peak(device, ms, ctypes.byref(v)))
    return v.value


from . import workloads  # noqa: E402,F401  (config builders)
