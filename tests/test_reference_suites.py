"""Drop-in proof: the reference's own C++ suites (proj/tests/*.cpp, compiled
unchanged by tests/cpp/Makefile against this framework's headers and
libqk_b200.so, with a doctest-subset shim) run and pass.

Host-only suites (gates, circuit text, tools/generators) run on the CPU; the
engine, distributed, optimizer (fidelity checks), CLI and acceptance suites
need the B200.  The one expected failure is the reference's kernel-backend
selection case (test_engine.cpp:322-331): this framework has no CPU backends
to select (the north star forbids multi-backend dispatch)."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "tests", "cpp", "_bin")
EXPECTED_FAILURES = {"test_engine": {"kernel backend selection validates its argument"}}


def run_suite(name, timeout=1200):
    path = os.path.join(BIN, name)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (make -C tests/cpp where /root/reference exists)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=timeout, cwd=BIN)
    failed = set(re.findall(r"^FAILED TEST CASE: (.*) \(", r.stdout, re.M))
    return r, failed


@pytest.mark.parametrize("name", ["test_gates", "test_circuit", "test_tools"])
def test_host_suites(name):
    r, failed = run_suite(name)
    assert r.returncode == 0 and not failed, r.stdout[-3000:]
    assert "[doctest-subset]" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["test_engine", "test_distributed", "test_optimizer", "test_cli"])
def test_device_suites(name):
    r, failed = run_suite(name)
    assert "[doctest-subset]" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]
    assert failed <= EXPECTED_FAILURES.get(name, set()), r.stdout[-4000:]


@pytest.mark.gpu
def test_acceptance():
    r, _ = run_suite("acceptance")
    fails = [ln for ln in r.stdout.splitlines() if ln.startswith("FAIL:")]
    assert not fails and r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
