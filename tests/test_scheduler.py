"""Host scheduler (CPU): the pass programs compiled for a block, replayed by
the numpy kernel emulator (tests/emulator.py), reproduce the reference's
applyBlock (the plain-C oracle) — register maps, deferred diagonal factors,
X relabels, exchanges and multi-CTA tiles are all exercised without a GPU."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from emulator import run_steps
from oracle import config_text

P = json.load(open(os.path.join(GOLDEN, "golden_programs.json")))
G = np.load(os.path.join(GOLDEN, "golden_states.npz"))


def emulate(qk, lines, n, st):
    out = st.view(np.complex128).copy()
    run_steps(out, n, qk.debug_compile_block(lines, n))
    return out


@pytest.mark.parametrize("name", ["mixed", "random5_0", "random5_1", "random5_2"])
def test_golden_blocks(qk, name):
    case = P[f"block/{name}"]
    got = emulate(qk, case["lines"], case["n"], G[f"block/{name}/in"])
    assert np.max(np.abs(got - G[f"block/{name}/out"].view(np.complex128))) < 1e-12


@pytest.mark.parametrize("n,chunk", [(4, 4), (6, 3), (9, 9), (11, 7), (13, 13), (14, 12)])
def test_random_blocks(qk, port, n, chunk):
    rng = np.random.default_rng(n * 31 + chunk)
    for seed in range(3):
        lines = [ln for ln in qk.generate("random", chunk, 80, 1000 * n + seed).splitlines() if ln.strip()]
        st = rng.standard_normal(2 << n)
        want = st.copy()
        port.apply_block(want, n, lines, chunk)
        assert np.max(np.abs(emulate(qk, lines, n, st) - want.view(np.complex128))) < 1e-12, seed


def test_x_heavy_sequences(qk, port):
    # X relabels interleaved with every other kind (flipped slots everywhere)
    n = 11
    rng = np.random.default_rng(5)
    kinds = ["H", "X", "U", "RZ", "CP", "RZZ", "CX", "SWAP", "RX"]
    for trial in range(6):
        lines = []
        for gid in range(60):
            k = kinds[int(rng.integers(len(kinds)))] if gid % 3 else "X"
            q = [int(x) for x in rng.choice(n, 2, replace=False)]
            if k in ("H", "X"):
                lines.append(f"{k} {q[0]} {gid}")
            elif k in ("RZ", "RX"):
                lines.append(f"{k} {q[0]} {gid} {rng.normal():.6f}")
            elif k == "U":
                lines.append(f"U {q[0]} {gid} 0.3 {rng.normal():.6f} -0.2")
            elif k in ("CP", "RZZ"):
                lines.append(f"{k} {q[0]} {q[1]} {gid} {rng.normal():.6f}")
            else:
                lines.append(f"{k} {q[0]} {q[1]} {gid}")
        st = rng.standard_normal(2 << n)
        want = st.copy()
        port.apply_block(want, n, lines, n)
        assert np.max(np.abs(emulate(qk, lines, n, st) - want.view(np.complex128))) < 1e-12, trial


@pytest.mark.parametrize("f", [2, 3, 4, 5])
def test_fused_blocks(qk, port, ref, f):
    n = 10
    for kind, a in (("qaoa", 2), ("random", 90), ("qft", 0), ("bvones", 0)):
        prog = ref.optimize(ref.gen(kind, n, a, 17), config_text(n, 0, 8, f))
        lines = prog.splitlines()
        i = 0
        rng = np.random.default_rng(f)
        while i < len(lines):
            k = int(lines[i])
            body = lines[i + 1:i + 1 + k]
            i += 1 + k
            if body[0].startswith("SQS"):
                continue
            st = rng.standard_normal(2 << n)
            want = st.copy()
            port.apply_block(want, n, body, 8)
            assert np.max(np.abs(emulate(qk, body, n, st) - want.view(np.complex128))) < 1e-11, kind


def test_pass_capacity_split(qk, port):
    # > kMaxOps gates in one block: the scheduler splits into several passes
    n = 9
    lines = [ln for ln in qk.generate("random", n, 1500, 3).splitlines() if ln.strip()]
    prog = qk.debug_compile_block(lines, n)
    assert len(prog["steps"]) >= 2
    st = np.random.default_rng(1).standard_normal(2 << n)
    want = st.copy()
    port.apply_block(want, n, lines, n)
    out = st.view(np.complex128).copy()
    run_steps(out, n, prog)
    assert np.max(np.abs(out - want.view(np.complex128))) < 1e-11


def run_compiled(qk, port, prog, n, initial):
    """Replay the engine's compiled item list (lazy IMS included) on the CPU.
    The run starts in the compiled initial layout mem0 (program position p at
    memory bit mem0[p]); identity unless compiled for a basis-state run."""
    compiled = prog.debug_compile(n)
    st = np.zeros(1 << n, dtype=np.complex128)
    st[sum(((initial >> p) & 1) << m for p, m in enumerate(compiled["mem0"]))] = 1
    for it in compiled["items"]:
        if it["kind"] == 0:
            run_steps(st, n, it["block"])
        elif it["kind"] == 1:
            f = st.view(np.float64)
            port.ims_swap(f, n, [tuple(p) for p in it["pairs"]])
        else:
            raise AssertionError("cross-rank item in a single-rank program")
    return st


@pytest.mark.parametrize("name", sorted(k for k in P if "program" in P[k] and P[k]["r"] == 0))
def test_compiled_programs_match_golden(qk, port, name):
    case = P[name]
    prog = qk.Program.parse(case["program"], qk.Config.parse(case["config"]))
    for initial in (0, 5):
        got = run_compiled(qk, port, prog, case["n"], initial)
        want = G[f"{name}/init{initial}/state"].view(np.complex128)
        assert np.max(np.abs(got - want)) < 1e-10


@pytest.mark.parametrize("name", sorted(k for k in P if "program" in P[k] and P[k]["r"] == 0))
def test_free_initial_layout_programs_match_golden(qk, port, name, monkeypatch):
    # compiled as qk_simulate compiles them (run from a basis state): the
    # slice starts in the layout that ends the first stream in physical order
    monkeypatch.setenv("QK_DEBUG_FROM_BASIS", "1")
    case = P[name]
    prog = qk.Program.parse(case["program"], qk.Config.parse(case["config"]))
    for initial in (0, 5):
        got = run_compiled(qk, port, prog, case["n"], initial)
        want = G[f"{name}/init{initial}/state"].view(np.complex128)
        assert np.max(np.abs(got - want)) < 1e-10


def test_free_initial_layout_needs_no_materialization(qk, monkeypatch):
    monkeypatch.setenv("QK_DEBUG_FROM_BASIS", "1")
    n = 16
    cfg = qk.Config.make(n, 0, chunk=8, fusion=0, diag=0)
    prog = qk.Program.optimize(qk.generate("qft", n), cfg)
    compiled = prog.debug_compile()
    assert prog.counts()["sqs"] > 2 and not [it for it in compiled["items"] if it["kind"] == 1]
    assert sorted(compiled["mem0"]) == list(range(n)) and compiled["mem0"] != list(range(n))


def test_lazy_ims_removes_swap_passes(qk):
    n = 16
    cfg = qk.Config.make(n, 0, chunk=8, fusion=0, diag=0)
    prog = qk.Program.optimize(qk.generate("qft", n), cfg)
    items = prog.debug_compile()["items"]
    ims = [it for it in items if it["kind"] == 1]
    assert prog.counts()["sqs"] > 2 and len(ims) <= 2  # only the final materialization


def test_random_programs_lazy(qk, port, ref):
    rng = np.random.default_rng(77)
    for i in range(12):
        n = int(rng.integers(5, 11))
        c = int(rng.integers(3, n + 1))
        cfg_text = config_text(n, 0, c, fusion=i % 2, diag=(i // 2) % 2)
        circ = ref.gen("random", n, 70, 500 + i)
        prog_text = ref.optimize(circ, cfg_text)
        want, _, _, _ = ref.simulate(prog_text, cfg_text, n, 0, 3, 1)
        prog = qk.Program.parse(prog_text, qk.Config.parse(cfg_text))
        got = run_compiled(qk, port, prog, n, 3)
        assert np.max(np.abs(got - want.view(np.complex128))) < 1e-10, i


def test_specialized_kernel_sources_compile(qk):
    # generator output is valid CUDA for sm_100a (NVRTC runs without a GPU)
    mixed = ["H 0 0", "X 2 1", "U 1 2 0.3 1.1 -0.7", "RX 3 3 0.9", "RY 0 4 -1.3", "RZ 2 5 2.2",
             "RZZ 1 3 6 0.8", "CP 0 3 7 1.9", "CX 3 1 8", "CX 0 2 9", "SWAP 1 2 10", "CP 3 0 11 -0.6"]
    src = qk.debug_jit_compile(mixed, 9)
    assert "__global__" in src and "switch" not in src
    prog = qk.Program.optimize(qk.generate("qaoa", 12, 1, 3), qk.Config.make(12, 0, chunk=8, fusion_qubits=3))
    lines = prog.text().splitlines()
    k = int(lines[0])
    assert qk.debug_jit_compile(lines[1:1 + k], 14)


@pytest.mark.parametrize("seed", range(6))
def test_streams_with_out_of_tile_diagonals(qk, port, ref, seed):
    # n > 13: passes span program blocks and apply diagonal gates whose qubits
    # lie outside the tile (CTA-constant bits: per-CTA factors, D_k CTA offsets).
    n = 15
    rng = np.random.default_rng(seed)
    kind = ["qft", "qaoa", "random"][seed % 3]
    circ = ref.gen(kind, n, {"qft": 0, "qaoa": 1, "random": 150}[kind], 40 + seed)
    cfg_text = config_text(n, 0, int(rng.integers(5, 11)), fusion=seed % 2, diag=(seed // 2) % 2)
    prog_text = ref.optimize(circ, cfg_text)
    want, _, _, _ = ref.simulate(prog_text, cfg_text, n, 0, 9, 2)
    prog = qk.Program.parse(prog_text, qk.Config.parse(cfg_text))
    compiled = prog.debug_compile()
    got = run_compiled(qk, port, prog, n, 9)
    assert np.max(np.abs(got - want.view(np.complex128))) < 1e-10
    if kind == "qft":
        assert any(s.get("ncta", 0) > 0 for it in compiled["items"] if it["kind"] == 0 for s in it["block"]["steps"])


@pytest.mark.parametrize("n", [1, 2, 3])
def test_tiny_programs_compile(qk, port, ref, n):
    # slices under 4 qubits run every gate as a dense group (no routing)
    cfg_text = config_text(n, 0, n, fusion=0, diag=0)
    prog_text = ref.optimize(ref.gen("random", n, 25, 40 + n), cfg_text)
    prog = qk.Program.parse(prog_text, qk.Config.parse(cfg_text))
    want, _, _, _ = ref.simulate(prog_text, cfg_text, n, 0, 1, 1)
    got = run_compiled(qk, port, prog, n, 1)
    assert np.max(np.abs(got - want.view(np.complex128))) < 1e-12


def toffoli_lines(a, b, t, gid):
    """The 15-gate H / T / CX Toffoli (Grover's AND chain, csrc/host/tools.cpp)."""
    q = 0.78539816339744828
    seq = [("H", t), ("CX", b, t), ("U", t, -q), ("CX", a, t), ("U", t, q), ("CX", b, t), ("U", t, -q),
           ("CX", a, t), ("U", b, q), ("U", t, q), ("H", t), ("CX", a, b), ("U", a, q), ("U", b, -q), ("CX", a, b)]
    out = []
    for g in seq:
        if g[0] == "H":
            out.append(f"H {g[1]} {gid}")
        elif g[0] == "CX":
            out.append(f"CX {g[1]} {g[2]} {gid}")
        else:
            out.append(f"U {g[1]} {gid} 0 0 {g[2]!r}")
        gid += 1
    return out, gid


def toffoli_circuit(n, count, seed):
    """Toffolis on random triples, X flips (control polarities), H and RZ
    between them (partial overlaps end a fusion window), as circuit text."""
    rng = np.random.default_rng(seed)
    lines, gid = [f"H {q} {q}" for q in range(n)], n
    for _ in range(count):
        a, b, t = (int(x) for x in rng.choice(n, 3, replace=False))
        for q in rng.choice(n, 2, replace=False):
            lines.append(f"X {int(q)} {gid}")
            gid += 1
        tl, gid = toffoli_lines(a, b, t, gid)
        lines += tl
        if rng.random() < 0.5:
            lines.append(f"RZ {int(rng.integers(n))} {gid} {rng.normal():.6f}")
            gid += 1
        if rng.random() < 0.3:
            lines.append(f"H {int(rng.integers(n))} {gid}")
            gid += 1
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("n,chunk,seed", [(6, 6, 0), (9, 5, 1), (11, 8, 2), (14, 13, 3), (15, 9, 4)])
def test_toffoli_fusion(qk, port, ref, n, chunk, seed):
    # fuseToffolis: each 15-gate Toffoli becomes one OP_CCX (controls in
    # register slots or thread bits, either polarity) -- results vs the
    # reference's gate-by-gate simulateProgram
    cfg_text = config_text(n, 0, chunk, fusion=0, diag=0)
    prog_text = ref.optimize(toffoli_circuit(n, 12, seed), cfg_text)
    want, _, _, _ = ref.simulate(prog_text, cfg_text, n, 0, 3, 1)
    prog = qk.Program.parse(prog_text, qk.Config.parse(cfg_text))
    ops = [o[0] for it in prog.debug_compile(n)["items"] if it["kind"] == 0
           for s in it["block"]["steps"] if s["kind"] == 0 for o in s["ops"]]
    assert ops.count(24) >= 6  # OP_CCX
    got = run_compiled(qk, port, prog, n, 3)
    assert np.max(np.abs(got - want.view(np.complex128))) < 1e-10


def test_toffoli_fusion_grover(qk, port):
    # Grover's oracle + diffusion (AND chain of Toffolis into ancillas) vs the
    # plain-C oracle replaying the same program gate by gate
    n = 14
    cfg = qk.Config.make(n, 0, chunk=10, fusion=0, diag=0)
    prog = qk.Program.optimize(qk.generate("grover", n, 2, 5), cfg)
    ops = [o[0] for it in prog.debug_compile(n)["items"] if it["kind"] == 0
           for s in it["block"]["steps"] if s["kind"] == 0 for o in s["ops"]]
    assert ops.count(24) >= 20
    got = run_compiled(qk, port, prog, n, 6)
    want = port.run_program(prog.text(), n, 10, 6).view(np.complex128)
    assert np.max(np.abs(got - want)) < 1e-10


@pytest.mark.parametrize("kind,n,seed", [("toffoli", 16, 11), ("toffoli", 17, 12), ("bvones", 17, 0), ("random", 16, 13)])
def test_cta_bit_controls(qk, port, ref, kind, n, seed):
    # CX / CCX controls outside the pass's tile (QK_CTA_CONTROLS): selects on
    # the CTA's base index; only the target must be in the tile
    cfg_text = config_text(n, 0, 6, fusion=0, diag=0)
    circ = toffoli_circuit(n, 16, seed) if kind == "toffoli" else ref.gen(kind, n, 200 if kind == "random" else 0, seed)
    prog_text = ref.optimize(circ, cfg_text)
    want, _, _, _ = ref.simulate(prog_text, cfg_text, n, 0, 9, 1)
    prog = qk.Program.parse(prog_text, qk.Config.parse(cfg_text))
    ops = [o for it in prog.debug_compile(n)["items"] if it["kind"] == 0
           for s in it["block"]["steps"] if s["kind"] == 0 for o in s["ops"]]
    assert sum(1 for o in ops if (o[0] == 2 and o[3] & 4) or (o[0] == 24 and o[3] & 48)) >= (2 if kind == "toffoli" else 0)
    got = run_compiled(qk, port, prog, n, 9)
    assert np.max(np.abs(got - want.view(np.complex128))) < 1e-10
