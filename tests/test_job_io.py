"""Job files / results CSV / CLI on the GPU backend,
against the reference's own job_io (ref src/job_io.cpp):

* tests/cpp/test_job_io.cpp mirrors the reference's tests/test_job_io.cpp;
* cross-reads with the reference itself (oracle/_ref, build container only):
  the reference reads our job files, and our results CSV survives the
  reference's read_results + write_results byte for byte (byte-compatible
  17-digit format);
* the `mcb` CLI end to end: gen-fig1 -> run -> check-fig1 (acceptance
  criterion 1 through the files, on the GPU)."""
import os
import subprocess
import sys

import pytest

from tests import _oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "_build", "test_job_io")
CLI = os.path.join(ROOT, "paper_2104_10073_b200", "mcb")


def build():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    libdir = os.path.join(ROOT, "paper_2104_10073_b200")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_job_io.cpp"),
                    os.path.join(libdir, "libmcb.so"), "-Wl,-rpath," + libdir, "-o", EXE], check=True)
    return EXE


def test_job_io_cpu_cases(tmp_path):
    r = subprocess.run([build(), "cpu", str(tmp_path)], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    ref = _oracle.load_ref()
    if ref is None:
        return  # the cross-reads need the reference build (build container)
    # the reference reads our job file (strict nlohmann reader, unknown fields rejected)
    out = tmp_path / "ref_rewritten_job.json"
    n = ref.ref_job_roundtrip(str(tmp_path / "fig1_job.json").encode(), str(out).encode())
    assert n == 100, ref.ref_last_error()
    n = ref.ref_job_roundtrip(str(tmp_path / "roundtrip_job.json").encode(), str(out).encode())
    assert n == 3, ref.ref_last_error()
    # ... and we read the reference's serialisation of it
    import paper_2104_10073_b200  # noqa: F401  (library must be loadable)
    # our CSV survives the reference's reader + writer byte for byte
    ours = tmp_path / "roundtrip_results.csv"
    theirs = tmp_path / "ref_rewritten_results.csv"
    assert ref.ref_results_roundtrip(str(ours).encode(), str(theirs).encode()) == 6
    assert ours.read_bytes() == theirs.read_bytes()


def test_cli_usage_and_validate(tmp_path):
    assert os.path.exists(CLI), "build the CLI: make -C paper_2104_10073_b200/csrc"
    r = subprocess.run([CLI], capture_output=True, text=True)
    assert r.returncode == 2 and "usage" in r.stderr
    job = tmp_path / "job.json"
    assert subprocess.run([CLI, "gen-fig1", "--n", "12", "--samples", "1000", "--out", str(job)]).returncode == 0
    r = subprocess.run([CLI, "validate", str(job)], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.strip() == "ok: 12 integrand(s)"
    bad = tmp_path / "bad.json"
    bad.write_text('{"seed":1,"trials":1,"integrands":[{"name":"a","expr":"x3","dim":2,'
                   '"low":[0,0],"high":[1,1],"samples":100}]}')
    r = subprocess.run([CLI, "validate", str(bad)], capture_output=True, text=True)
    assert r.returncode == 2 and "a: x3 exceeds dim=2" in r.stderr


@pytest.mark.gpu
def test_job_io_run_command_on_gpu(gpu, tmp_path):
    r = subprocess.run([build(), "gpu", str(tmp_path)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cli_fig1_end_to_end(gpu, tmp_path):
    """acceptance.cpp criterion 1 through the files: gen-fig1 (100 x 1e6 x 10),
    run, check-fig1 >= 95/100 inside the 4-sigma band."""
    job, res, plot = tmp_path / "fig1.json", tmp_path / "fig1.csv", tmp_path / "plot.csv"
    assert subprocess.run([CLI, "gen-fig1", "--out", str(job)]).returncode == 0
    r = subprocess.run([CLI, "run", str(job), "--out", str(res)], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr
    assert r.stdout.count("\n") == 100 and r.stdout.startswith("f001: ")
    r = subprocess.run([CLI, "check-fig1", str(res), "--plot-out", str(plot)], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stdout[-2000:]
    passed = int(r.stdout.strip().splitlines()[-1].split()[1].split("/")[0])
    assert passed >= 95
    assert plot.read_text().startswith("n,mean,trial_stddev,analytic\n")
    # the reference reads our results file when available (build container)
    ref = _oracle.load_ref()
    if ref is not None:
        assert ref.ref_results_roundtrip(str(res).encode(), str(tmp_path / "x.csv").encode()) == 100
