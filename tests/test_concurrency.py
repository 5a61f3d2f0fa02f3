"""Concurrent callers of the C-ABI (ctypes releases the GIL around foreign
calls): every entry point serialises per device on its context (stream,
buffers, pinned staging), the JIT cache and the tree rounds are shared
state, and error messages are per thread — so N threads issuing mixed
calls at once must get exactly the bytes a sequential run gets."""
import threading

import numpy as np
import pytest


def _workloads(mcb):
    from paper_2104_10073_b200 import workloads as w
    harm = list(w.c1(60_000)[0][:6])
    strat = [mcb.stratify(f) for f in w.c1(50_000)[0][6:10]]
    peak = mcb.Program("exp(-a*((x1-0.5)^2+(x2-0.4)^2)) + x1", 2, ["a"])
    progs = [peak.integrand({"a": 10.0 + i}, n_samples=40_000, index=20 + i) for i in range(3)]
    trees = [mcb.tree(peak.integrand({"a": 30.0}, n_samples=60_000, index=30), samples_per_cell=500)]
    return [("direct", harm, 3), ("stratified", strat, 2), ("programs", progs, 2), ("tree", trees, 2),
            ("mixed", harm[:2] + strat[:1] + progs[:1] + trees, 2)], peak


@pytest.mark.gpu
def test_concurrent_run_direct_matches_sequential(gpu):
    cases, keep = _workloads(gpu)
    want = {name: gpu.run_direct(fns, 4242, trials).tobytes() for name, fns, trials in cases}
    got, errors = {}, []
    lock = threading.Lock()

    def worker(tid):
        try:
            for rep in range(3):
                name, fns, trials = cases[(tid + rep) % len(cases)]
                out = gpu.run_direct(fns, 4242, trials, devices=[0] if tid % 2 else [0, 0])
                with lock:
                    got.setdefault(name, []).append(out.tobytes())
        except Exception as e:  # surfaced below
            with lock:
                errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(6)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    assert sum(len(v) for v in got.values()) == 18
    for name, outs in got.items():
        assert all(o == want[name] for o in outs), name
    del keep


@pytest.mark.gpu
def test_errors_are_per_thread(gpu):
    """A failing call in one thread does not clobber another thread's
    mcb_last_error, and successful calls keep running alongside."""
    from paper_2104_10073_b200 import workloads as w
    good = list(w.c1(20_000)[0][:2])
    bad = gpu.harmonic(1.0, 4, n_samples=1000)
    bad.low[0], bad.high[0] = 1.0, 0.0  # empty domain: validation error
    msgs, ok = [], []

    def failing():
        for _ in range(20):
            try:
                gpu.run_direct([bad], 1, 2)
            except Exception as e:
                msgs.append(str(e))

    def passing():
        for _ in range(20):
            ok.append(gpu.run_direct(good, 1, 2).tobytes())

    ts = [threading.Thread(target=failing), threading.Thread(target=passing)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert len(msgs) == 20 and all(m == msgs[0] for m in msgs) and msgs[0]
    assert len(set(ok)) == 1
