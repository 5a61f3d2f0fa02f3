"""Multi-process (N > 1) host logic on the CPU with the gloo backend,
world_size 2: weak-scaling shards (bench.py), the max-over-ranks timing
reduction, and LPT device sharding covering every integrand exactly once
(mcb_partition).  The data path has no collective: only the final timing
reduction crosses ranks."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench
    import paper_2104_10073_b200 as mcb
    from paper_2104_10073_b200 import workloads

    d = bench.Dist(world, rank, "gloo")
    first = bench.shard_first_index(rank, 1000)
    fns, _, _ = workloads.c2(samples=1000, n_count=1000, first_index=first)
    idx = [f.integrand_index for f in fns]
    # per-rank timing -> max over ranks
    t = 1.0 + rank
    tmax = d.max(t)
    # device sharding inside one process (mcb_run_direct's LPT)
    shards = mcb.partition(fns, 10, 4)
    d.barrier()
    d.close()
    out_q.put((rank, idx[0], idx[-1], len(set(idx)), tmax, np.bincount(shards, minlength=4).tolist()))


def test_weak_scaling_shards_and_max_over_ranks():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, a0, b0, n0, t0, s0), (r1, a1, b1, n1, t1, s1) = res
    # disjoint global integrand ranges -> disjoint Philox keys, no exchange needed
    assert (a0, b0, n0) == (0, 999, 1000) and (a1, b1, n1) == (1000, 1999, 1000)
    assert t0 == t1 == 2.0
    assert sum(s0) == 1000 and max(s0) - min(s0) <= 1


def test_partition_covers_each_integrand_once():
    import paper_2104_10073_b200 as mcb
    from paper_2104_10073_b200 import workloads
    fns, _, _ = workloads.c5(samples=10_000_000, n_fns=2000)
    for n in (1, 2, 4, 8):
        s = mcb.partition(fns, 10, n)
        assert s.min() == 0 and s.max() == n - 1 and len(s) == len(fns)
        # cost balance within 1% (LPT on n_samples * trials * per-sample cost)
        cost = np.zeros(n)
        per = {mcb.FAMILY_ABS2: 1.2, mcb.FAMILY_ABS3: 1.7}
        for f, k in zip(fns, s):
            c = per.get(f.family, 0.5 * f.dim + 1.0)
            cost[k] += c
        assert cost.max() / cost.mean() < 1.01


def test_reference_arm_json_contract():
    """bench.py --impl reference prints one JSON line (CPU only; tiny sample)."""
    ref_so = os.path.join(ROOT, "oracle", "_ref", "libmcbatch_ref.so")
    env = dict(os.environ)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0", "--samples", "20000", "--cpu-seconds", "1"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "cpu_baseline", "e2e", "config", "higher_is_better"):
        assert k in line
    assert line["cpu_baseline"]["kind"] == ("reference" if os.path.exists(ref_so) else "port")
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["value"] > 0


def test_strong_scaling_slices_cover_the_set_once():
    import bench
    for world in (1, 2, 3, 4, 8):
        seen = []
        for rank in range(world):
            lo, hi = bench.strong_slice(1000, rank, world)
            seen.extend(range(lo, hi))
        assert seen == list(range(1000))
