"""The C++ host API (include/mcb/mcbatch.hpp) exercised by a compiled test
program that mirrors the reference's own doctest suites case by case
(tests/cpp/test_mcbatch.cpp).  Compilation is checked on the CPU; running it
needs the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "_build", "test_mcbatch")


def build():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    libdir = os.path.join(ROOT, "paper_2104_10073_b200")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_mcbatch.cpp"),
                    os.path.join(libdir, "libmcb.so"), "-Wl,-rpath," + libdir, "-o", EXE],
                   check=True)
    return EXE


def test_cpp_api_compiles_against_header_and_library():
    assert os.path.exists(build())


@pytest.mark.gpu
def test_cpp_api_suite_on_gpu(gpu):
    exe = build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
