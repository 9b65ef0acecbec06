"""The quokka_b200 CLI drop-in (proj/tools/main.cpp subcommands): same text
outputs and exit codes as the reference CLI (tests/test_cli.cpp scenarios)."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from oracle import config_text

CLI = os.path.join(ROOT, "paper_2409_14697_b200", "quokka_b200")


def run(*args, cwd=None):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, cwd=cwd, timeout=300)


def test_gen_matches_reference(ref, tmp_path):
    for which, extra, kind, a, seed in (("qft", [], "qft", 0, 0), ("qaoa", ["-l", "2", "--seed", "7"], "qaoa", 2, 7),
                                        ("random", ["-g", "50", "--seed", "3"], "random", 50, 3),
                                        ("bv", [], "bvones", 0, 0)):
        r = run("gen", which, "-n", 9, *extra)
        assert r.returncode == 0, r.stderr
        assert r.stdout == ref.gen(kind, 9, a, seed)


def test_optimize_forms_match_reference(ref, tmp_path):
    circ = tmp_path / "c.txt"
    circ.write_text(ref.gen("qft", 10))
    cfg = tmp_path / "cfg.ini"
    cfg.write_text(config_text(10, 0, 5))
    r1 = run("optimize", "-i", circ, "--config", cfg)
    r2 = run("optimize", circ, 5, 10, 10, 1, 1, 5, 1)  # positional finder form
    assert r1.returncode == 0 and r2.returncode == 0
    assert r1.stdout == ref.optimize(ref.gen("qft", 10), config_text(10, 0, 5))
    assert r1.stdout == r2.stdout


def test_exit_codes(tmp_path):
    assert run("simulate", "-i", "nope.ini").returncode == 2             # bad command line
    assert run("optimize", tmp_path / "missing.txt", 5, 10, 10, 1, 1, 5, 1).returncode == 1  # unreadable input
    bad = tmp_path / "bad.txt"
    bad.write_text("FOO 1 2\n")
    assert run("optimize", bad, 5, 10, 10, 1, 1, 5, 1).returncode == 1   # ParseError
    assert run("gen", "nosuch", "-n", 5).returncode == 2                 # ConfigError


@pytest.mark.gpu
def test_simulate_dump_state_matches_oracle(ref, tmp_path):
    n = 12
    for kind, a, seed, r in (("qft", 0, 0, 0), ("random", 60, 4, 0), ("qaoa", 1, 2, 1)):
        circ_text = ref.gen(kind, n, a, seed)
        cfg = tmp_path / "cfg.ini"
        cfg.write_text(config_text(n, r, 6, b=n - r - 1))
        prog = tmp_path / "p.txt"
        prog.write_text(ref.optimize(circ_text, config_text(n, r, 6, b=n - r - 1)))
        out = run("simulate", "-i", cfg, "-c", prog, "--dump-state", "--initial", 3)
        assert out.returncode == 0, out.stderr
        lines = out.stdout.splitlines()
        assert lines[0] == f"qubits: {n}" and lines[1].startswith("gates: ") and lines[3].startswith("norm: ")
        amps = np.array([[float(x) for x in ln.split()[1:]] for ln in lines[4:]])
        got = amps[:, 0] + 1j * amps[:, 1]
        want = ref.oracle_simulate(circ_text, n, 3).view(np.complex128)
        assert np.max(np.abs(got - want)) < 1e-10, kind
        assert abs(float(lines[3].split()[1]) - 1.0) < 1e-12
