"""Test configuration.

Markers: ``gpu`` — needs a B200 (sm_100a); everything else runs on the CPU.
The oracle (oracle/mcb_oracle.c) is the checker; it is built here on demand
with gcc if its .so is missing (test infrastructure only)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU (sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from tests import _oracle
    return _oracle.load()


@pytest.fixture(scope="session")
def mcb():
    import paper_2104_10073_b200 as m
    return m


@pytest.fixture(scope="session")
def gpu(mcb):
    if mcb.device_count() < 1:
        pytest.fail("no CUDA device visible: -m gpu tests need a B200 (no CPU fallback exists)")
    return mcb


def pytest_terminal_summary(terminalreporter):
    """Largest deviation / tolerance per parity comparison (tests/_deviation.py)."""
    from tests import _deviation
    lines = _deviation.summary_lines()
    if lines:
        terminalreporter.write_sep("-", "parity margins: max |gpu - ref| / tolerance")
        for line in lines:
            terminalreporter.write_line(line)
