"""Drop-in proof: the reference's own C++ suites (proj/tests/*.cpp, compiled
unchanged by tests/cpp/Makefile against this framework's headers and
libqk_b200.so, with a doctest-subset shim) run and pass.

Host-only suites (gates, circuit text, tools/generators) run on the CPU; the
engine, distributed, optimizer (fidelity checks), CLI and acceptance suites
need the B200.  The expected failures are listed (and justified) in
EXPECTED_FAILURES below."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "tests", "cpp", "_bin")
# Two reference cases test properties of its CPU kernels, not of the result:
#  * backend selection (test_engine.cpp:322-331): there is no CPU backend to
#    select here (the north star forbids multi-backend dispatch);
#  * "applyBlock equals gate-by-gate application bit for bit"
#    (test_engine.cpp:210-233): the reference applies each gate of a block
#    with the same scalar kernel as applyGate, so the two agree bitwise; the
#    fused pass kernels here reassociate (H scales folded into one power of
#    two, diagonal phases deferred and batched), so blocks agree with
#    gate-by-gate application to ~1e-16 per amplitude, not bitwise
#    (tests/test_gpu_kernels.py holds blocks to 1e-12 against the reference).
EXPECTED_FAILURES = {"test_engine": {"kernel backend selection validates its argument",
                                     "applyBlock equals gate-by-gate application bit for bit"}}


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
