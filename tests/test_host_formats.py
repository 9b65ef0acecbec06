"""Host layer parity (CPU): text formats, generators and the AIO optimizer of
the product library are byte-identical to the reference
(proj/src/circuit.cpp, tools.cpp, optimizer.cpp) and to the golden fixtures."""
import json
import os

import pytest

from conftest import GOLDEN
from oracle import config_text

P = json.load(open(os.path.join(GOLDEN, "golden_programs.json")))

GEN_CASES = [("qft", 13, 0, 0), ("qft", 31, 0, 0), ("qaoa", 9, 2, 11), ("qaoa", 31, 5, 1),
             ("bv", 9, 0, 0b10110101), ("bvones", 31, 0, 0), ("random", 12, 150, 7),
             ("random", 1, 10, 3), ("bench:U", 7, 0, 0), ("bench:RZZ", 6, 0, 0), ("bench:CP", 5, 0, 0)]


@pytest.mark.parametrize("kind,n,a,seed", GEN_CASES)
def test_generators_match_reference(ref, qk, kind, n, a, seed):
    assert qk.generate(kind, n, a, seed) == ref.gen(kind, n, a, seed)


def test_generator_counts(qk):
    # proj/tests/acceptance.cpp:147-155: 496 / 2511 / 92 gates.
    assert len(qk.generate("qft", 31).splitlines()) == 496
    assert len(qk.generate("qaoa", 31, 5, 1).splitlines()) == 2511
    assert len(qk.generate("bvones", 31).splitlines()) == 92


@pytest.mark.parametrize("name", sorted(k for k in P if "program" in P[k]))
def test_optimizer_matches_golden(qk, name):
    case = P[name]
    cfg = qk.Config.parse(case["config"])
    assert qk.Program.optimize(case["circuit"], cfg).text() == case["program"]


def test_optimizer_matches_reference_random(ref, qk):
    # acceptance.cpp:67-96 style sweep: random circuits x flag combinations x ranks.
    import numpy as np
    rng = np.random.default_rng(9000)
    for i in range(120):
        n = int(rng.integers(4, 13))
        gates = int(rng.integers(10, 61))
        r = i % 3
        c = min(3 + int(rng.integers(0, 3)), n - r)
        flags = i % 16
        cfg_text = config_text(n, r, c, ims=flags & 1, xrs=(flags >> 1) & 1, fusion=(flags >> 2) & 1,
                               diag=(flags >> 3) & 1)
        circ = ref.gen("random", n, gates, 31000 + i)
        try:
            want = ref.optimize(circ, cfg_text)
        except Exception as e:  # same error class expected
            with pytest.raises(qk.QuokkaError) as ei:
                qk.Program.optimize(circ, qk.Config.parse(cfg_text))
            assert ei.value.code == e.code
            continue
        got = qk.Program.optimize(circ, qk.Config.parse(cfg_text)).text()
        assert got == want, (i, n, r, c, flags)


def test_showcase_structure(qk):
    # proj/tests/test_optimizer.cpp:297-328 (unfused) and :330-366 (fused).
    case = P["showcase_plain"]
    prog = qk.Program.optimize(case["circuit"], qk.Config.parse(case["config"]))
    assert prog.counts() == {"blocks": 4, "sqs": 5, "csqs": 1, "gates": 14}
    swaps = [ln for ln in prog.text().splitlines() if ln.startswith(("SQS", "CSQS"))]
    assert swaps == ["SQS 3 0 1 2 5 6 7", "SQS 3 0 1 3 4 5 7", "SQS 1 5 6", "CSQS 2 6 7 8 9",
                     "SQS 1 5 6", "SQS 3 0 2 3 5 6 7"]
    fused = qk.Program.optimize(case["circuit"], qk.Config.parse(P["showcase_fused"]["config"])).text()
    dl = [ln.split() for ln in fused.splitlines() if ln.startswith("D4")]
    assert [d[5:7] for d in dl] == [["0.75390225434330471", "-0.65698659871878906"],
                                    ["-0.83907152907645244", "0.54402111088936966"]]


def test_qft31_within_twenty_blocks(qk):
    cfg = qk.Config.make(31, 0, chunk=10, fusion=0, diag=0)
    assert qk.Program.optimize(qk.generate("qft", 31), cfg).counts()["blocks"] <= 20


def test_program_roundtrip_matches_reference(ref, qk):
    for name, case in P.items():
        if "program" not in case:
            continue
        cfg = qk.Config.parse(case["config"])
        assert qk.Program.parse(case["program"], cfg).text() == ref.program_roundtrip(case["program"], case["config"])
    # bare swap lines (circuit.cpp:414-437) and lenient parsing
    cfg_t = config_text(6, 1, 3)
    text = "1\nH 0 0\nSQS 1 0 4\n1\nCSQS 1 2 5\n"
    assert qk.Program.parse(text, qk.Config.parse(cfg_t)).text() == ref.program_roundtrip(text, cfg_t)
    wide = "1\nH 5 0\n"
    assert qk.Program.parse(wide, qk.Config.parse(cfg_t), lenient=True).text() == \
        ref.program_roundtrip(wide, cfg_t, lenient=True)


def test_circuit_and_config_roundtrip(ref, qk):
    text = "H 0 0 # c\nCX 1 0 1\nU 2 2 0.1 0.2 0.3 // x\nCP 0 2 3 1e-3\nRZZ 1 2 4 -2.5\nSWAP 0 1 5\nRZ 2 6\n"
    assert qk.circuit_roundtrip(text) == ref.circuit_roundtrip(text)
    ini = "# cfg\n[system]\ntotal_qbit = 12\nrank_qbit=2\nchunk_qbit=5\nfusion=0\n"
    assert qk.Config.parse(ini).text() == ref.config_roundtrip(ini)


@pytest.mark.parametrize("bad,code", [
    ("H 0\n", 1), ("FOO 0 0\n", 1), ("CX 0 0 1\n", 1), ("H 0 0\nH 1 0\n", 1), ("D2 0 1 1 0\n", 1),
    ("RX 0 0 0.1 0.2\n", 1), ("H -1 0\n", 1),
])
def test_circuit_errors_match_reference(ref, qk, bad, code):
    with pytest.raises(qk.QuokkaError) as ei:
        qk.circuit_roundtrip(bad)
    assert ei.value.code == code
    from oracle import RefError
    with pytest.raises(RefError) as er:
        ref.circuit_roundtrip(bad)
    assert er.value.code == code


@pytest.mark.parametrize("ini", [
    "[system]\nrank_qbit=1\n", "[system]\ntotal_qbit=41\n", "[other]\ntotal_qbit=4\n",
    "[system]\ntotal_qbit=8\nchunk_qbit=9\n", "[system]\ntotal_qbit=8\nfoo=1\n",
    "[system]\ntotal_qbit=x\n", "[system]\ntotal_qbit=6\nrank_qbit=6\n",
])
def test_config_errors(qk, ini):
    with pytest.raises(qk.ConfigError):
        qk.Config.parse(ini)


@pytest.mark.parametrize("prog", [
    "2\nH 0 0\n", "1\nH 4 0\n", "SQS 2 0 1 2\n", "SQS 1 0 6\n", "CSQS 1 0 2\n", "SQS 2 1 0 2 3\n",
    "1 2\nH 0 0\n", "2\nH 0 0\nSQS 1 0 1\n",
])
def test_program_errors(ref, qk, prog):
    cfg_t = config_text(6, 1, 3)
    with pytest.raises(qk.ParseError):
        qk.Program.parse(prog, qk.Config.parse(cfg_t))
    from oracle import RefError
    with pytest.raises(RefError):
        ref.program_roundtrip(prog, cfg_t)
