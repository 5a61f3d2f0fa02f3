"""The GPU Philox of the fused kernels against cuRAND's independent
curand_Philox4x32_10 on the device: 2^20 random
(key, chunk, trial, block) counters, bit-exact (tests/cpp/test_curand_philox.cu)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_curand_philox.cu")
EXE = os.path.join(ROOT, "tests", "cpp", "_build", "test_curand_philox")


def build():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17",
                    "-I" + os.path.join(ROOT, "paper_2104_10073_b200", "csrc"), "-I" + os.path.join(ROOT, "include"),
                    SRC, "-o", EXE], check=True)
    return EXE


def test_curand_cross_check_builds():
    assert os.path.exists(build())


@pytest.mark.gpu
def test_philox_matches_curand_on_gpu(gpu):
    exe = EXE if os.path.exists(EXE) else build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0 and " 0 mismatches" in r.stdout, r.stdout + r.stderr
