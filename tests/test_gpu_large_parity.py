"""Parity at the sizes and code paths the bench and BASELINE.json's configs run.

* QFT-30 (BASELINE config 2) in both program forms the reference produces:
  the GPU-tuned one bench.py times (chunk_qbit 13, fusion off) and the
  reference-default fused one (chunk_qbit 10, fusion_qbit 5, D_k diagonal
  fusion) -- against the closed form of genQft|x>.
* BV with fusion_qbit 5: every fused U5 runs on the wide dense-group path --
  against the BV closed form (tools.cpp:199-216).
* QAOA-28 / random-28 (400 gates) at chunk_qbit 13, unfused, against the
  reference's own simulateProgram (oracle/_ref) amplitude by amplitude.
* IMS at 27 qubits, where both IMS kernels take several trips per thread /
  warp (the incremental GF(2) walks): bit-exact against bitswap on an
  index-encoded state (engine.cpp:86-101).
* The reference optimizer's fused programs at 26 qubits (U5 tiles, D_k
  tables, IMS) from a nonzero basis state vs its simulateProgram.

Tolerance: 1e-10 max abs per amplitude, |norm - 1| < 1e-12 (north star);
permutations bit-exact.
"""
import numpy as np
import pytest

from oracle import config_text
from test_gpu_programs import TOL, qft_expected

pytestmark = pytest.mark.gpu


def logical_to_phys(p2l):
    l2p = {l: p for p, l in enumerate(p2l)}
    return lambda logical: sum(((logical >> l) & 1) << l2p[l] for l in range(len(p2l)))


def check_qft_windows(st, n, x, p2l, window=1 << 20):
    rng = np.random.default_rng(n)
    for off in (0, (1 << n) - window, int(rng.integers(0, (1 << n) - window)) & ~(window - 1)):
        got = st.download(off, window)
        want = qft_expected(n, x, p2l, np.arange(off, off + window, dtype=np.int64))
        assert np.max(np.abs(got - want)) < TOL, off
    assert abs(st.norm() - 1.0) < 1e-12


@pytest.mark.parametrize("form", ["bench", "reference_default"])
def test_qft30_closed_form(qk, form):
    n = 30
    if form == "bench":
        cfg = qk.Config.make(n, 0, chunk=13, fusion=0, diag=0)
    else:
        cfg = qk.Config.make(n, 0)  # chunk 10, fusion 5, diagonal fusion: D_k up to D10
    prog = qk.Program.optimize(qk.generate("qft", n), cfg)
    if form == "reference_default":
        assert "D10 " in prog.text()
    x = 0x2C3B5A1D & ((1 << n) - 1)
    st = qk.State(n)
    try:
        for _ in range(2):  # first run times the autotune variants, second runs the choice
            st.simulate(prog, x)
            check_qft_windows(st, n, x, prog.final_layout())
    finally:
        st.close()


@pytest.mark.parametrize("n,chunk", [(30, 13), (30, 10), (33, 13)])
def test_bv_fused_u5_closed_form(qk, n, chunk):
    cfg = qk.Config.make(n, 0, chunk=chunk, fusion_qubits=5)
    prog = qk.Program.optimize(qk.generate("bvones", n), cfg)
    assert "U5 " in prog.text()
    st = qk.State(n)
    try:
        st.simulate(prog, 0)
        phys = logical_to_phys(prog.final_layout())
        secret = (1 << (n - 1)) - 1
        a = st.download(phys(secret), 1)[0]
        b = st.download(phys(secret | (1 << (n - 1))), 1)[0]
        assert abs(a - 1 / np.sqrt(2)) < TOL and abs(b + 1 / np.sqrt(2)) < TOL
        assert abs(st.norm() - 1.0) < 1e-12  # all other amplitudes are 0
        rng = np.random.default_rng(n)
        for off in rng.integers(0, (1 << n) - 4096, 4):
            w = st.download(int(off), 4096)
            idx = np.arange(int(off), int(off) + 4096)
            mask = (idx != phys(secret)) & (idx != phys(secret | (1 << (n - 1))))
            assert np.max(np.abs(w[mask])) < TOL
    finally:
        st.close()


@pytest.mark.parametrize("kind,a,seed", [("qaoa", 1, 1), ("random", 400, 7)])
def test_28q_vs_reference(ref, qk, kind, a, seed):
    n = 28
    cfg_text = config_text(n, 0, 13, fusion=0, diag=0)
    prog_text = ref.optimize(ref.gen(kind, n, a, seed), cfg_text)
    initial = 0x5A5A5A5 & ((1 << n) - 1)
    want, wl, _, _ = ref.simulate(prog_text, cfg_text, n, 0, initial, 0)
    want = want.view(np.complex128)
    prog = qk.Program.parse(prog_text, qk.Config.parse(cfg_text))
    st = qk.State(n)
    try:
        for run in range(3):  # autotune: the 2^13 / 2^12-tile schedules and register widths all run
            st.simulate(prog, initial)
            step = 1 << 24
            for off in range(0, 1 << n, step):
                got = st.download(off, step)
                assert np.max(np.abs(got - want[off:off + step])) < TOL, (run, off)
        assert prog.final_layout() == wl
        assert abs(st.norm() - 1.0) < 1e-12
    finally:
        st.close()


def bitswap_np(x, pairs):
    for o, i in pairs:
        d = ((x >> o) ^ (x >> i)) & 1
        x = x ^ ((d << o) | (d << i))
    return x


@pytest.mark.parametrize("mode", [0, 1])
def test_ims_multi_trip_bitexact(qk, mode):
    # n = 27: k_ims walks 2^7 elements per thread, k_ims_tiled 2^(n-k-16)
    # orbits per warp, so their incremental GF(2) steps are exercised.
    n = 27
    idx = np.arange(1 << n, dtype=np.int64)
    host = np.empty(1 << n, dtype=np.complex128)
    host.real = idx
    host.imag = -idx
    st = qk.State(n)
    pair_sets = [[(0, 26)], [(0, 20), (1, 25), (2, 13)], [(3, 24), (5, 22), (9, 26)],
                 [(0, 1)], [(1, 2), (4, 23), (6, 21), (7, 19), (8, 26)], [(20, 26), (21, 25), (22, 24)]]
    try:
        qk.set_ims_mode(mode)
        for pairs in pair_sets:
            st.upload(host)
            qk.ims_swap(st, pairs)
            got = st.download()
            src = bitswap_np(idx, pairs)  # a[bitswap(i)] <- a[i], an involution
            assert np.array_equal(got.real, src.astype(np.float64)), pairs
            assert np.array_equal(got.imag, -src.astype(np.float64)), pairs
    finally:
        qk.set_ims_mode(1)
        st.close()


@pytest.mark.parametrize("kind,a,seed,flags", [("random", 300, 11, dict()),                     # reference defaults: U5 + D_k
                                               ("qaoa", 2, 4, dict(c=12)),                      # D_k fusion, chunk 12
                                               ("qft", 0, 0, dict(c=11, fusion=0, diag=1))])   # D_k only
def test_26q_reference_default_flags(ref, qk, kind, a, seed, flags):
    # the reference optimizer's fused programs (U5 tile kernel, D_k tables,
    # IMS materializations) from a nonzero basis state, amplitude by
    # amplitude against the reference's simulateProgram
    n = 26
    flags = dict(flags)
    c = flags.pop("c", None)
    cfg_text = config_text(n, 0, c, **flags)
    prog_text = ref.optimize(ref.gen(kind, n, a, seed), cfg_text)
    initial = 0x2B3C4D5 & ((1 << n) - 1)
    want, wl, _, _ = ref.simulate(prog_text, cfg_text, n, 0, initial, 0)
    want = want.view(np.complex128)
    prog = qk.Program.parse(prog_text, qk.Config.parse(cfg_text))
    st = qk.State(n)
    try:
        for run in range(2):
            st.simulate(prog, initial)
            got = st.download()
            assert np.max(np.abs(got - want)) < TOL, run
        assert prog.final_layout() == wl
        assert abs(st.norm() - 1.0) < 1e-12
    finally:
        st.close()
