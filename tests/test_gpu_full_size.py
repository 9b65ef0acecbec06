"""BASELINE.json's single-GPU sizes (2^33 amplitudes = 128 GiB in HBM): the
CPU oracle cannot hold them, so these check closed-form amplitudes (SURVEY
§8c KATs) on sampled windows, and the norm to 1e-12.  Programs are the ones
bench.py times (reference optimizer output, chunk_qbit 13, fusion off)."""
import numpy as np
import pytest

from test_gpu_programs import TOL, qft_expected

pytestmark = pytest.mark.gpu
N = 33


def program(qk, kind, a=0, seed=0):
    cfg = qk.Config.make(N, 0, chunk=13, fusion=0, diag=0)
    return qk.Program.optimize(qk.generate(kind, N, a, seed), cfg)


def logical_to_phys(p2l):
    l2p = {l: p for p, l in enumerate(p2l)}
    return lambda logical: sum(((logical >> l) & 1) << l2p[l] for l in range(len(p2l)))


def test_qft33_closed_form(qk):
    prog = program(qk, "qft")
    x = 0x1_2C3B_5A1D & ((1 << N) - 1)
    st = qk.State(N)
    try:
        st.simulate(prog, x)
        p2l = prog.final_layout()
        rng = np.random.default_rng(33)
        for off in (0, (1 << N) - (1 << 18), int(rng.integers(0, (1 << N) - (1 << 18)))):
            got = st.download(off, 1 << 18)
            want = qft_expected(N, x, p2l, np.arange(off, off + (1 << 18), dtype=np.int64))
            assert np.max(np.abs(got - want)) < TOL
        assert abs(st.norm() - 1.0) < 1e-12
    finally:
        st.close()


def test_grover33_closed_form(qk):
    m = (N + 2) // 2  # 17 data qubits, 16 ancillas
    marked, iters = 5, 1
    prog = program(qk, "grover", iters, marked)
    st = qk.State(N)
    try:
        st.simulate(prog, 0)
        phys = logical_to_phys(prog.final_layout())
        th = np.arcsin(2 ** (-m / 2))
        sign = (-1) ** iters
        amp = lambda logical: st.download(phys(logical), 1)[0]  # noqa: E731
        assert abs(amp(marked) - sign * np.sin((2 * iters + 1) * th)) < TOL
        other = sign * np.cos((2 * iters + 1) * th) / np.sqrt(2 ** m - 1)
        rng = np.random.default_rng(5)
        for d in rng.integers(0, 1 << m, 64):
            if int(d) != marked:
                assert abs(amp(int(d)) - other) < TOL
        for anc in rng.integers(1, 1 << (N - m), 32):  # ancillas back at |0>
            assert abs(amp((int(anc) << m) | int(rng.integers(0, 1 << m)))) < TOL
        assert abs(st.norm() - 1.0) < 1e-12
    finally:
        st.close()


def test_bv33_closed_form(qk):
    prog = program(qk, "bvones")
    st = qk.State(N)
    try:
        st.simulate(prog, 0)
        phys = logical_to_phys(prog.final_layout())
        secret = (1 << (N - 1)) - 1
        a = st.download(phys(secret), 1)[0]
        b = st.download(phys(secret | (1 << (N - 1))), 1)[0]
        assert abs(a - 1 / np.sqrt(2)) < TOL and abs(b + 1 / np.sqrt(2)) < TOL
        assert abs(st.norm() - 1.0) < 1e-12
    finally:
        st.close()
