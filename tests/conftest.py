"""Shared fixtures.  `gpu` marks tests that need a CUDA B200 (run with -m gpu)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


def _ensure_built():
    lib = os.path.join(ROOT, "paper_2409_14697_b200", "libqk_b200.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_2409_14697_b200")], check=True)
    oracle_lib = os.path.join(ROOT, "oracle", "_ref", "libqk_oracle.so")
    if not os.path.exists(oracle_lib):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


_ensure_built()


@pytest.fixture(scope="session")
def ref():
    """The reference build (oracle/_ref/libquokka_ref.so)."""
    from oracle import Ref
    path = os.path.join(ROOT, "oracle", "_ref", "libquokka_ref.so")
    if not os.path.exists(path):
        pytest.skip("reference build not present (built by `make -C oracle` where /root/reference exists)")
    return Ref()


@pytest.fixture(scope="session")
def port():
    """The plain-C restatement (oracle/quokka_oracle.c)."""
    from oracle import Port
    return Port()


@pytest.fixture(scope="session")
def qk():
    import paper_2409_14697_b200 as m
    return m
