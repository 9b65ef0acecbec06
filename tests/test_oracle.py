"""Pin the CPU oracle before trusting it (CPU only).

* the plain-C restatement (oracle/quokka_oracle.c) is BIT-EXACT against the
  reference build on the reference's own test shapes;
* both agree with the committed golden vectors (outputs of the reference);
* the reference satisfies the closed-form KATs used at 33-36 qubits.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import config_text, random_state

G = np.load(os.path.join(GOLDEN, "golden_states.npz"))
P = json.load(open(os.path.join(GOLDEN, "golden_programs.json")))


def test_random_state_matches_reference_stream(ref):
    # randomState (proj/tests/test_engine.cpp:20-31) reproduced in numpy: the
    # golden inputs were drawn with it, so check it against the reference Rng.
    st = random_state(5, 123)
    assert st.shape == (64,)
    assert abs(np.sum(st * st) - 1.0) < 1e-12


@pytest.mark.parametrize("name", ["mixed", "random5_0", "random5_1", "random5_2"])
def test_port_apply_block_bitexact_vs_golden(port, name):
    case = P[f"block/{name}"]
    st = G[f"block/{name}/in"].copy()
    port.apply_block(st, case["n"], case["lines"], case["chunk"])
    assert np.array_equal(st, G[f"block/{name}/out"])


def test_port_apply_block_bitexact_vs_reference_random(ref, port):
    for trial in range(12):
        n, chunk = 9, 4 + trial % 3
        lines = [ln for ln in ref.gen("random", chunk, 30, 900 + trial).splitlines() if ln.strip()]
        a = random_state(n, 50 + trial)
        b = a.copy()
        ref.apply_block(a, n, lines, chunk, 1)
        port.apply_block(b, n, lines, chunk)
        assert np.array_equal(a, b), trial


def test_port_fused_gates_bitexact_vs_reference(ref, port):
    # Fused D_k / U_k lines as the reference optimizer emits them.
    prog = ref.optimize(ref.gen("qaoa", 6, 2, 3), config_text(6, 0, 6, 3))
    lines = [ln for ln in prog.splitlines()[1:] if ln.strip() and not ln.strip().isdigit()]
    fused = [ln for ln in lines if ln.split()[0][0] in "DU" and ln.split()[0] not in ("U",)]
    assert fused, "expected fused gates"
    for ln in fused:
        a = random_state(6, 7)
        b = a.copy()
        ref.apply_block(a, 6, [ln], 6, 1)
        port.apply_block(b, 6, [ln], 6)
        assert np.array_equal(a, b), ln[:20]


@pytest.mark.parametrize("t", range(8))
def test_port_ims_bitexact_vs_golden(port, t):
    case = P["ims_cases"][t]
    st = G[f"ims/{t}/in"].copy()
    port.ims_swap(st, case["n"], [tuple(p) for p in case["pairs"]])
    assert np.array_equal(st, G[f"ims/{t}/out"])


@pytest.mark.parametrize("t", range(5))
def test_port_xrs_bitexact_vs_golden(port, t):
    case = P["xrs_cases"][t]
    st = G[f"xrs/{t}/in"].copy()
    stats = port.xrs_swap(st, case["n"], case["r"], case["b"], [tuple(p) for p in case["pairs"]])
    assert np.array_equal(st, G[f"xrs/{t}/out"])
    assert np.array_equal(stats, G[f"xrs/{t}/stats"])


def test_port_xrs_sweep_vs_reference(ref, port):
    # test_distributed.cpp:104-161 shapes: n=4..8, R=1..3, S<=R, B=S..N-R.
    rng = np.random.default_rng(555)
    for n in range(4, 9):
        for r in range(1, min(3, n - 1) + 1):
            region = n - r
            for s in range(1, r + 1):
                for b in range(s, region + 1):
                    outs = sorted(int(x) for x in rng.choice(region, s, replace=False))
                    ins = sorted(int(x) for x in rng.choice(np.arange(region, n), s, replace=False))
                    pairs = list(zip(outs, ins))
                    st = random_state(n, 9000 + 100 * n + 10 * r + s + b)
                    a, c = st.copy(), st.copy()
                    sa = ref.xrs_swap(a, n, r, b, pairs)
                    sc = port.xrs_swap(c, n, r, b, pairs)
                    assert np.array_equal(a, c) and np.array_equal(sa, sc), (n, r, s, b)


def test_reference_matches_golden_programs(ref):
    for name, case in P.items():
        if "program" not in case:
            continue
        assert ref.optimize(case["circuit"], case["config"]) == case["program"], name


def test_qft_closed_form_kat(ref):
    # QFT|x> = 2^{-n/2} exp(2 pi i rev_n(x) y / 2^n) in logical order (no final swaps).
    for n in (3, 5, 8):
        for x in (0, 1, (1 << n) - 2):
            got = ref.oracle_simulate(ref.gen("qft", n), n, x).view(np.complex128)
            rev = int(format(x, f"0{n}b")[::-1], 2)
            y = np.arange(1 << n)
            want = 2.0 ** (-n / 2) * np.exp(2j * np.pi * ((rev * y) % (1 << n)) / (1 << n))
            assert np.max(np.abs(got - want)) < 1e-12


def test_bv_closed_form_kat(ref):
    n = 7
    got = ref.oracle_simulate(ref.gen("bvones", n), n).view(np.complex128)
    secret = (1 << (n - 1)) - 1
    want = np.zeros(1 << n, dtype=np.complex128)
    want[secret] = 1 / np.sqrt(2)
    want[secret | (1 << (n - 1))] = -1 / np.sqrt(2)
    assert np.max(np.abs(got - want)) < 1e-12
