"""Straight-line specialized pass kernels (jit.cpp) vs the oracle and vs the
pass interpreter, on every gate kind, fused gates, flips and multi-segment
passes.  The threshold is forced to 0 so small slices exercise them."""
import numpy as np
import pytest

from oracle import config_text, random_state

pytestmark = pytest.mark.gpu


@pytest.fixture()
def jit(qk):
    qk.set_jit_min_qubits(0)
    yield qk
    qk.set_jit_min_qubits(22)


def run(qk, st, n, lines, chunk):
    d = qk.State(n)
    d.upload(st.view(np.complex128))
    qk.apply_block(d, lines, chunk)
    out = d.download()
    d.close()
    return out


@pytest.mark.parametrize("n,chunk", [(4, 4), (7, 5), (9, 9), (12, 10), (13, 13), (14, 13), (16, 12)])
def test_random_blocks(ref, jit, n, chunk):
    for seed in range(3):
        lines = [ln for ln in ref.gen("random", chunk, 80, 70 * n + seed).splitlines() if ln.strip()]
        st = np.random.default_rng(seed).standard_normal(2 << n)
        want = st.copy()
        ref.apply_block(want, n, lines, chunk, 4)
        assert np.max(np.abs(run(jit, st, n, lines, chunk) - want.view(np.complex128))) < 1e-12, seed


@pytest.mark.parametrize("kind", ["H", "U", "X", "RX", "RY", "RZ", "CX", "CP", "SWAP", "RZZ"])
def test_every_kind(ref, jit, kind):
    n = 14
    st = np.random.default_rng(3).standard_normal(2 << n)
    lines = [ln for ln in ref.gen(f"bench:{kind}", n).splitlines() if ln.strip()]
    want = st.copy()
    ref.apply_block(want, n, lines, n, 4)
    assert np.max(np.abs(run(jit, st, n, lines, n) - want.view(np.complex128))) < 1e-12


@pytest.mark.parametrize("f", [2, 3, 4, 5])
def test_fused_programs(ref, jit, f):
    n = 13
    for kind, a in (("qaoa", 2), ("random", 150), ("qft", 0), ("bvones", 0)):
        cfg_text = config_text(n, 0, 9, f)
        prog = ref.optimize(ref.gen(kind, n, a, 21), cfg_text)
        want, wl, _, _ = ref.simulate(prog, cfg_text, n, 0, 77, 4)
        p = jit.Program.parse(prog, jit.Config.parse(cfg_text))
        st, p2l = jit.simulate_program(p, 77)
        assert np.max(np.abs(st - want.view(np.complex128))) < 1e-10, kind
        assert p2l == wl


def test_qft_matches_interpreter(qk):
    n = 24
    cfg = qk.Config.make(n, 0, chunk=13, fusion=0, diag=0)
    prog = qk.Program.optimize(qk.generate("qft", n), cfg)
    qk.set_jit_min_qubits(-1)
    a, _ = qk.simulate_program(prog, 12345)
    qk.set_jit_min_qubits(0)
    b, _ = qk.simulate_program(prog, 12345)
    qk.set_jit_min_qubits(22)
    assert np.max(np.abs(a - b)) < 1e-13
