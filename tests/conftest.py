"""Test configuration.

Markers: ``gpu`` = needs a B200 (run with ``-m gpu`` on the GPU box); everything
else runs on CPU.  The oracle (oracle/, test infrastructure) is built on demand.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle_py
    return oracle_py.oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle_py
    if not oracle_py.ref_available():
        pytest.skip("oracle/_ref (reference build) not present")
    return oracle_py.ref()


@pytest.fixture(scope="session")
def ss():
    """The product package with its CUDA library built (build() if missing)."""
    lib = os.path.join(ROOT, "paper_2111_11866_b200", "libsubsurf_b200.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2111_11866_b200", "csrc"), "-s", "-j8"],
                       check=True)
    import paper_2111_11866_b200 as m
    return m


@pytest.fixture(scope="session")
def gpu(ss):
    if not ss.device_available():
        pytest.fail("no CUDA device: " + ss.library().ss_last_error().decode())
    return ss
