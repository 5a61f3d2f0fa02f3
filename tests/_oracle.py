"""ctypes view of the CPU oracle (oracle/mcb_oracle.c) — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may use this module, and only as the checker.  Built with gcc
on demand (oracle/Makefile) when the .so is missing."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "_build", "libmcb_oracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libmcbatch_ref.so")

_lib = None


class ChunkAccum(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint64), ("n_nonfinite", ctypes.c_uint64),
                ("mean", ctypes.c_double), ("m2", ctypes.c_double)]


def build() -> str:
    # make tracks mcb_oracle.c and include/mcb/mcb.h (the shared struct layouts)
    subprocess.run(["make", "-s", "-C", ORACLE_DIR, "all"], check=True)
    return ORACLE_SO


def load():
    global _lib
    if _lib is not None:
        return _lib
    from paper_2104_10073_b200 import Integrand, Leaf, TrialStats  # struct layouts only
    build()
    lib = ctypes.CDLL(ORACLE_SO)
    P = ctypes.POINTER
    u32, u64, dbl, i32, vp, sz = (ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double, ctypes.c_int,
                                  ctypes.c_void_p, ctypes.c_size_t)
    sig = {
        "orc_splitmix64": (u64, [u64]),
        "orc_stream_key": (None, [u64, u32, P(u32)]),
        "orc_philox4x32_10": (None, [P(u32), P(u32), P(u32)]),
        "orc_to_unit_double": (dbl, [u32, u32]),
        "orc_sample_uniform": (i32, [u32, P(dbl), P(dbl), u64, u32, u32, u64, u64, u64, vp]),
        "orc_eval": (dbl, [P(Integrand), P(dbl)]),
        "orc_accum_add": (None, [P(ChunkAccum), dbl]),
        "orc_accum_merge": (None, [P(ChunkAccum), P(ChunkAccum)]),
        "orc_accumulate_chunk": (i32, [P(Integrand), u64, u32, u64, u64, P(ChunkAccum)]),
        "orc_volume": (dbl, [P(Integrand)]),
        "orc_chunk_count": (u64, [u64]),
        "orc_direct_mc": (i32, [P(Integrand), u64, u32, u64, P(TrialStats)]),
        "orc_summarize_trials": (i32, [P(TrialStats), u32, P(dbl), P(dbl), P(u32)]),
        "orc_run_direct": (i32, [P(Integrand), sz, u64, u32, i32, vp]),
        "orc_harmonic_k": (dbl, [u32]),
        "orc_stratified_mc": (i32, [P(Integrand), u64, u32, u64, P(TrialStats)]),
        "orc_stratified_plan": (i32, [P(Integrand), P(u32), P(u64), P(u32)]),
        "orc_grid_cell": (None, [P(Integrand), u32, u64, P(dbl), P(dbl)]),
        "orc_harmonic_closed_form": (dbl, [dbl, u32]),
        "orc_tree_refine": (i32, [P(Integrand), u64, u32, u64, P(TrialStats), P(Leaf), sz, P(sz)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def philox(ctr, key):
    lib = load()
    out = (ctypes.c_uint32 * 4)()
    lib.orc_philox4x32_10((ctypes.c_uint32 * 4)(*ctr), (ctypes.c_uint32 * 2)(*key), out)
    return [int(v) for v in out]


def stream_key(seed, index):
    lib = load()
    k = (ctypes.c_uint32 * 2)()
    lib.orc_stream_key(seed, index, k)
    return int(k[0]), int(k[1])


def sample_uniform(low, high, seed, integrand, trial, chunk, first_point, count):
    lib = load()
    d = len(low)
    out = np.zeros((count, d), dtype=np.float64)
    rc = lib.orc_sample_uniform(d, (ctypes.c_double * d)(*low), (ctypes.c_double * d)(*high), seed,
                                integrand, trial, chunk, first_point, count, out.ctypes.data)
    if rc != 0:
        raise ValueError("invalid domain or chunk")
    return out


def eval_points(f, pts):
    lib = load()
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    out = np.empty(len(pts))
    row = (ctypes.c_double * 8)()
    for i in range(len(pts)):
        for j in range(pts.shape[1]):
            row[j] = pts[i, j]
        out[i] = lib.orc_eval(ctypes.byref(f), row)
    return out


def tree_refine(f, seed, trial=0, chunk_base=0):
    """orc_tree_refine: (TrialStats, [Leaf]) — ref src/estimator.cpp:212-318."""
    from paper_2104_10073_b200 import Leaf, TrialStats
    lib = load()
    st = TrialStats()
    n = ctypes.c_size_t()
    if lib.orc_tree_refine(ctypes.byref(f), seed, trial, chunk_base, ctypes.byref(st), None, 0,
                           ctypes.byref(n)) != 0:
        raise ValueError("oracle tree_refine failed")
    buf = (Leaf * max(1, n.value))()
    lib.orc_tree_refine(ctypes.byref(f), seed, trial, chunk_base, ctypes.byref(st), buf, n.value,
                        ctypes.byref(n))
    return st, list(buf[:n.value])


def ref_tree_refine(source, f, params, seed, trial=0, chunk_base=0):
    """The reference's own tree_refine of `source` (params: name -> value)."""
    from paper_2104_10073_b200 import Leaf, TrialStats
    lib = load_ref()
    if lib is None:
        raise FileNotFoundError(REF_SO)
    names = list(params)
    cn = (ctypes.c_char_p * max(1, len(names)))(*[n.encode() for n in names])
    cv = (ctypes.c_double * max(1, len(names)))(*[params[n] for n in names])
    st = TrialStats()
    n = ctypes.c_size_t()
    cap = 1 << 16
    buf = (Leaf * cap)()
    if lib.ref_tree_refine_source(source.encode(), ctypes.byref(f), cn, cv, len(names), seed, trial,
                                  chunk_base, ctypes.byref(st), buf, cap, ctypes.byref(n)) != 0:
        raise RuntimeError(lib.ref_last_error().decode())
    return st, list(buf[:min(n.value, cap)])


def ref_stratified_mc(source, f, params, cells_per_dim, spc, seed, trial=0, chunk_base=0, cell_cap=0):
    """The reference's own stratified_mc of `source` (params: name -> value)."""
    from paper_2104_10073_b200 import Leaf, TrialStats
    lib = load_ref()
    if lib is None:
        raise FileNotFoundError(REF_SO)
    names = list(params)
    cn = (ctypes.c_char_p * max(1, len(names)))(*[n.encode() for n in names])
    cv = (ctypes.c_double * max(1, len(names)))(*[params[n] for n in names])
    st = TrialStats()
    n = ctypes.c_size_t()
    cap = 1 << 16
    buf = (Leaf * cap)()
    if lib.ref_stratified_mc_source(source.encode(), ctypes.byref(f), cn, cv, len(names), cells_per_dim, spc,
                                    cell_cap, seed, trial, chunk_base, ctypes.byref(st), buf, cap,
                                    ctypes.byref(n)) != 0:
        raise RuntimeError(lib.ref_last_error().decode())
    return st, list(buf[:min(n.value, cap)])


def direct_mc(f, seed, trial=0, chunk_base=0):
    from paper_2104_10073_b200 import TrialStats
    lib = load()
    st = TrialStats()
    if lib.orc_direct_mc(ctypes.byref(f), seed, trial, chunk_base, ctypes.byref(st)) != 0:
        raise ValueError("oracle direct_mc failed")
    return st


def run_direct(fns, seed, trials, n_threads=None):
    from paper_2104_10073_b200 import TRIAL_DTYPE, as_array
    lib = load()
    arr = as_array(fns)
    out = np.zeros((len(arr), trials), dtype=TRIAL_DTYPE)
    n_threads = n_threads or os.cpu_count() or 1
    if lib.orc_run_direct(arr, len(arr), seed, trials, n_threads, out.ctypes.data) != 0:
        raise ValueError("oracle run_direct failed")
    return out


# ---- the reference itself, compiled from /root/reference sources (oracle/_ref) ----

_ref = None


def load_ref():
    """The unmodified reference library built by `make -C oracle ref` (None if absent)."""
    global _ref
    if _ref is not None:
        return _ref
    if not os.path.exists(REF_SO):
        return None
    from paper_2104_10073_b200 import Integrand, Leaf, TrialStats
    lib = ctypes.CDLL(REF_SO)
    P = ctypes.POINTER
    u32, u64, dbl, i32, sz = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double, ctypes.c_int, ctypes.c_size_t
    sig = {
        "ref_last_error": (ctypes.c_char_p, []),
        "ref_sample_uniform": (i32, [u32, P(dbl), P(dbl), u64, u32, u32, u64, u64, ctypes.c_void_p]),
        "ref_eval_points": (i32, [ctypes.c_char_p, P(Integrand), ctypes.c_void_p, u64, ctypes.c_void_p]),
        "ref_direct_mc": (i32, [ctypes.c_char_p, P(Integrand), u64, u32, u64, P(TrialStats)]),
        "ref_run_batch": (i32, [P(ctypes.c_char_p), P(Integrand), sz, u64, u32, u32, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, P(dbl)]),
        "ref_harmonic_job": (i32, [u32, u64, P(dbl), P(u64), P(u32)]),
        "ref_harmonic_closed_form": (dbl, [dbl]),
        "ref_eval_source": (i32, [ctypes.c_char_p, u32, P(ctypes.c_char_p), P(dbl), sz, ctypes.c_void_p, u64,
                                  ctypes.c_void_p]),
        "ref_direct_mc_source": (i32, [ctypes.c_char_p, u32, P(ctypes.c_char_p), P(dbl), sz, P(dbl), P(dbl),
                                       u64, u64, u32, u32, u64, P(TrialStats)]),
        "ref_analytic_harmonic": (dbl, [u32]),
        "ref_job_roundtrip": (i32, [ctypes.c_char_p, ctypes.c_char_p]),
        "ref_results_roundtrip": (i32, [ctypes.c_char_p, ctypes.c_char_p]),
        "ref_run_command": (i32, [ctypes.c_char_p, ctypes.c_char_p, i32]),
        "ref_stratified_mc_source": (i32, [ctypes.c_char_p, P(Integrand), P(ctypes.c_char_p), P(dbl), sz, u32, u32,
                                           u64, u64, u32, u64, P(TrialStats), P(Leaf), sz, P(sz)]),
        "ref_tree_refine_source": (i32, [ctypes.c_char_p, P(Integrand), P(ctypes.c_char_p), P(dbl), sz, u64,
                                         u32, u64, P(TrialStats), P(Leaf), sz, P(sz)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _ref = lib
    return lib


def ref_run_batch(fns, seed, trials, workers=0, sources=None):
    """run_batch of the unmodified reference on the lowered DSL sources (or
    `sources`: parameter-free DSL per integrand, for PROGRAM descriptors)."""
    from paper_2104_10073_b200 import TRIAL_DTYPE, as_array, to_dsl
    lib = load_ref()
    if lib is None:
        raise FileNotFoundError(REF_SO)
    arr = as_array(fns)
    n = len(arr)
    texts = sources if sources is not None else [to_dsl(arr[i]) for i in range(n)]
    srcs = (ctypes.c_char_p * n)(*[t.encode() for t in texts])
    out = np.zeros((n, trials), dtype=TRIAL_DTYPE)
    mean = np.zeros(n)
    sd = np.zeros(n)
    ok = np.zeros(n, dtype=np.int32)
    secs = ctypes.c_double()
    if lib.ref_run_batch(srcs, arr, n, seed, trials, workers, out.ctypes.data, mean.ctypes.data,
                         sd.ctypes.data, ok.ctypes.data, ctypes.byref(secs)) != 0:
        raise RuntimeError(lib.ref_last_error().decode())
    return out, mean, sd, ok, secs.value
