"""Host (CPU) build of the exact device arithmetic in mcb_device.cuh, checked
against the oracle: Philox with the CTA prefix, the exact 53-bit conversion,
the 2^-64 parameter folding, sincos accuracy and the quadrant-coefficient
identity (tests/cpp/test_device_math.cpp).  No GPU needed."""
import os
import subprocess

from tests import _oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_device_math_on_host():
    so = _oracle.build()
    out_dir = os.path.join(ROOT, "tests", "cpp", "_build")
    os.makedirs(out_dir, exist_ok=True)
    exe = os.path.join(out_dir, "test_device_math")
    subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off",
                    "-I" + os.path.join(ROOT, "paper_2104_10073_b200", "csrc"),
                    "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_device_math.cpp"), so,
                    "-Wl,-rpath," + os.path.dirname(so), "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
