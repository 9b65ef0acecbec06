"""The straight-line specialized pass kernels (jit.cpp's generated CUDA) run
on the CPU through tests/host/jit_host_shim.h — one std::thread per CUDA
thread, a std::barrier per __syncthreads — and must reproduce the reference
build on whole programs (lazy IMS, free output permutations, fused gates).
Catches generator bugs and intra-CTA load/store races without a GPU."""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

from jit_host import run_program_jit, run_program_jit_sparse
from oracle import config_text


@pytest.mark.parametrize("kind,n,chunk,fusion,diag,a,seed", [
    ("qft", 16, 13, 0, 0, 0, 0),      # single-segment last pass with a cross-thread store map
    ("qft", 15, 12, 0, 0, 0, 0),
    ("random", 14, 12, 1, 0, 160, 9),  # fused dense U_k
    ("qaoa", 14, 10, 1, 1, 1, 4),      # fused diagonals D_k
    ("bvones", 14, 13, 0, 0, 0, 0),
])
def test_specialized_kernels_on_host(ref, qk, port, kind, n, chunk, fusion, diag, a, seed):
    cfg_text = config_text(n, 0, chunk, fusion=fusion, diag=diag)
    prog_text = ref.optimize(ref.gen(kind, n, a, seed), cfg_text)
    want, _, _, _ = ref.simulate(prog_text, cfg_text, n, 0, 5, 2)
    prog = qk.Program.parse(prog_text, qk.Config.parse(cfg_text))
    st = np.zeros(1 << n, dtype=np.complex128)
    st[5] = 1
    run_program_jit(qk, port, prog, n, st)
    assert np.max(np.abs(st - want.view(np.complex128))) < 1e-10
    # folded initState: the first pass synthesizes |5> and never reads the slice
    st = np.full(1 << n, np.nan, dtype=np.complex128)
    run_program_jit(qk, port, prog, n, st, basis=5)
    assert np.max(np.abs(st - want.view(np.complex128))) < 1e-10


@pytest.mark.parametrize("rb", [4, 3])
def test_other_register_width_variants_on_host(rb):
    # QK_RB13=4 / 3: the register widths the runtime autotunes against
    # (16 / 8 amplitudes per thread, 512 / 1024 threads per 2^13 tile)
    code = r"""
import sys, numpy as np
sys.path[:0] = [%r, %r, %r]
import paper_2409_14697_b200 as qk
from oracle import Ref, Port, config_text
from jit_host import run_program_jit, run_program_jit_sparse
ref, port = Ref(), Port()
for kind, n, a in (("qft", 16, 0), ("random", 15, 150)):
    cfg_text = config_text(n, 0, 13, fusion=0, diag=0)
    pt = ref.optimize(ref.gen(kind, n, a, 3), cfg_text)
    want = ref.simulate(pt, cfg_text, n, 0, 5, 2)[0].view(np.complex128)
    prog = qk.Program.parse(pt, qk.Config.parse(cfg_text))
    assert all(s.get("rb") == RB for it in prog.debug_compile()["items"] if it["kind"] == 0
               for s in it["block"]["steps"] if s.get("ct") == 13)
    st = np.zeros(1 << n, dtype=np.complex128); st[5] = 1
    run_program_jit(qk, port, prog, n, st)
    assert np.max(np.abs(st - want)) < 1e-10, kind
print("ok")
""".replace("RB", str(rb)) % (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests"))
    env = dict(os.environ, QK_RB13=str(rb))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_tma_pipelined_kernels_on_host():
    # QK_JIT_TMA=1: 2^13 tiles with >= 128-B rows become persistent kernels
    # that stream the next tile into shared memory (cp.async.bulk + mbarrier)
    # and exchange in two halves.  Checked in a fresh process (the knob is
    # read once) on whole programs, against the reference build.
    code = r"""
import sys, numpy as np
sys.path[:0] = [%r, %r, %r]
import paper_2409_14697_b200 as qk
from oracle import Ref, Port, config_text
from jit_host import run_program_jit, run_program_jit_sparse
ref, port = Ref(), Port()
for kind, n, a in (("qft", 16, 0), ("qaoa", 15, 1)):
    cfg_text = config_text(n, 0, 13, fusion=0, diag=0)
    pt = ref.optimize(ref.gen(kind, n, a, 3), cfg_text)
    want = ref.simulate(pt, cfg_text, n, 0, 5, 2)[0].view(np.complex128)
    prog = qk.Program.parse(pt, qk.Config.parse(cfg_text))
    srcs = prog.debug_jit_sources()
    assert any("mbar_wait(mbar, phase)" in src for _, src in srcs), kind
    assert all(len(src) < 200_000 for _, src in srcs)  # linear-size code generation
    for basis in (None, 5):
        st = np.zeros(1 << n, dtype=np.complex128); st[5] = 1
        run_program_jit(qk, port, prog, n, st, basis=basis)
        assert np.max(np.abs(st - want)) < 1e-10, (kind, basis)
    # sparse start: support-only reads, output tiles through TMA bulk stores
    st = np.full(1 << n, np.nan, dtype=np.complex128)
    run_program_jit_sparse(qk, port, prog, n, st, 5)
    assert not np.isnan(st).any() and np.max(np.abs(st - want)) < 1e-10, (kind, "sparse")
print("ok")
""" % (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests"))
    env = dict(os.environ, QK_JIT_TMA="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("kind,n,a,seed", [("qft", 16, 0, 0), ("qaoa", 15, 1, 2), ("random", 15, 300, 4),
                                           ("bvones", 15, 0, 0)])
def test_sparse_start_on_host(ref, qk, port, kind, n, a, seed):
    # A run from a basis state as qk_simulate launches it: the basis pass
    # computes only its own tile (no memset -- the rest of the slice is NaN
    # here), later passes get the known-zero coset and skip what lies outside
    # it.  Any read of a never-written amplitude would show up as NaN.
    cfg_text = config_text(n, 0, 13, fusion=0, diag=0)
    prog_text = ref.optimize(ref.gen(kind, n, a, seed), cfg_text)
    want, _, _, _ = ref.simulate(prog_text, cfg_text, n, 0, 0x1235 & ((1 << n) - 1), 2)
    prog = qk.Program.parse(prog_text, qk.Config.parse(cfg_text))
    st = np.full(1 << n, np.nan, dtype=np.complex128)
    run_program_jit_sparse(qk, port, prog, n, st, 0x1235 & ((1 << n) - 1))
    assert not np.isnan(st).any()
    assert np.max(np.abs(st - want.view(np.complex128))) < 1e-10


@pytest.mark.parametrize("n,chunk,seed", [(14, 13, 3), (15, 11, 5)])
def test_toffoli_fusion_kernels_on_host(ref, qk, port, n, chunk, seed):
    # generated OP_CCX code (register renames and thread-bit selects) in the
    # specialized kernels, full and sparse-start runs, vs the reference
    from test_scheduler import toffoli_circuit
    cfg_text = config_text(n, 0, chunk, fusion=0, diag=0)
    prog_text = ref.optimize(toffoli_circuit(n, 14, seed), cfg_text)
    want, _, _, _ = ref.simulate(prog_text, cfg_text, n, 0, 5, 2)
    prog = qk.Program.parse(prog_text, qk.Config.parse(cfg_text))
    assert any("csel(c, y, x)" in src for _, src in prog.debug_jit_sources(n))
    st = np.zeros(1 << n, dtype=np.complex128)
    st[5] = 1
    run_program_jit(qk, port, prog, n, st)
    assert np.max(np.abs(st - want.view(np.complex128))) < 1e-10
    st = np.full(1 << n, np.nan, dtype=np.complex128)
    run_program_jit_sparse(qk, port, prog, n, st, 5)
    assert not np.isnan(st).any() and np.max(np.abs(st - want.view(np.complex128))) < 1e-10
