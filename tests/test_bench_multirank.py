"""bench.py's N > 1 path (torchrun, one process per rank, barrier + max over
ranks, rank 0 prints one JSON line) run on a one-GPU box: MCB_BENCH_SHARE_GPU=1
puts both ranks on the visible GPU over gloo.  The ranks compete for one GPU,
so only the contract is checked here, never the numbers."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(extra):
    env = dict(os.environ, MCB_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--samples", "100000", "--n-fns", "200",
           "--no-clocks", "--c5-fns", "64", "--c5-samples", "100000", *extra]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]  # rank 0 only
    return json.loads(lines[0])


@pytest.mark.gpu
@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_two_ranks(scaling):
    line = _torchrun(["--scaling", scaling])
    assert line["n_gpus"] == 2 and line["scaling"] == scaling and line["steps"] == 3
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
    assert line["roofline"]["frac"] > 0 and "cpu_baseline" not in line  # the CPU leg is rank 0 at N = 1 only
    # value = samples of all ranks per step / the slowest rank's step time
    per_step = (2 * 200 if scaling == "weak" else 200) * 100_000 * 10
    assert line["value"] * line["ms_per_step"] / 1e3 == pytest.approx(per_step, rel=1e-9)
    # e2e: rank 0 times the product's own scheduler over the whole job (both devices)
    assert "devices=[0, 0]" in line["e2e"]["path"]
    assert line["e2e"]["h2d_bytes_per_step"] == (2 * 200 if scaling == "weak" else 200) * 272
    # configs[4] (C5) weak and strong, max over ranks
    c5 = line["scaling_c5"]
    assert c5["weak"]["integrands"] == 2 * 8 and c5["strong"]["integrands"] == 64
    assert c5["weak"]["samples_per_s"] > 0 and c5["strong"]["samples_per_s"] > 0
    assert line["config"]["integrands"] == (400 if scaling == "weak" else 200)


def test_fused_roofline_arithmetic():
    import bench
    r = bench.fused_roofline(3.0e11, {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0})
    assert r["peak"] == pytest.approx(1.306 * 148 * 1.965e9 / 1e9)
    assert r["frac"] == pytest.approx(3.0e11 / (1.306 * 148 * 1.965e9))
    assert bench.fused_roofline(1.0, {"sm_mhz": None, "sm_max_mhz": None}) is None
