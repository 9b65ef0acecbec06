"""TEST INFRASTRUCTURE: compile the engine's generated specialized pass
kernels (jit.cpp) for the CPU with g++ through tests/host/jit_host_shim.h and
replay a compiled program with them, so the straight-line generator is
checked against the oracle without a GPU."""
import ctypes as C
import hashlib
import os
import subprocess

import numpy as np

from emulator import run_steps

HERE = os.path.dirname(os.path.abspath(__file__))
CACHE = os.path.join(HERE, ".jit_host_cache")


def host_kernel(name: str, src: str):
    os.makedirs(CACHE, exist_ok=True)
    body = src.replace("#include <cuda_runtime.h>", '#include "jit_host_shim.h"')
    body += f"\nQK_HOST_LAUNCHER({name})\n"
    h = hashlib.sha1(body.encode()).hexdigest()[:16]
    so = os.path.join(CACHE, f"{h}.so")
    if not os.path.exists(so):
        cpp = os.path.join(CACHE, f"{h}.cpp")
        open(cpp, "w").write(body)
        subprocess.run(["g++", "-std=c++20", "-O1", "-fPIC", "-shared", "-w", "-I", os.path.join(HERE, "host"),
                        cpp, "-o", so + ".tmp", "-lpthread"], check=True)
        os.replace(so + ".tmp", so)
    lib = C.CDLL(so)
    lib.qk_host_launch.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_uint64]
    lib.qk_host_launch2.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint,
                                    C.c_uint, C.c_uint64, C.c_uint64, C.c_uint]
    return lib.qk_host_launch if not sparse_launch else lib.qk_host_launch2


sparse_launch = False


def host_kernel2(name: str, src: str):
    global sparse_launch
    sparse_launch = True
    try:
        return host_kernel(name, src)
    finally:
        sparse_launch = False


NO_BASIS = (1 << 64) - 1


def run_program_jit(qk, port, prog, n_local, state, basis=None):
    """Replay prog's compiled items on `state` (complex128, 2^n_local) with the
    generated kernels for passes, the emulator for dense/diag-table steps and
    the oracle for IMS items.  basis: the first pass synthesizes |basis>
    instead of reading `state` (the engine's folded initState)."""
    first = NO_BASIS if basis is None else basis
    qk.set_jit_min_qubits(0)  # the schedule the specialized kernels run (the interpreter's differs)
    try:
        items = prog.debug_compile(n_local)["items"]
    finally:
        qk.set_jit_min_qubits(22)
    if basis is not None and not (items and items[0]["kind"] == 0 and items[0]["block"]["steps"][0]["kind"] == 0):
        state[:] = 0  # the engine folds initState only into a leading pass
        state[basis] = 1
        first = NO_BASIS
    srcs = iter(prog.debug_jit_sources(n_local))
    for it in items:
        if it["kind"] == 0:
            blk = it["block"]
            gt = np.array(blk["gtab"] if blk["gtab"] else [0.0, 0.0], dtype=np.float64)
            for st in blk["steps"]:
                if st["kind"] == 0:
                    name, src = next(srcs)
                    host_kernel(name, src)(state.ctypes.data, gt.ctypes.data, n_local, st["ct"], st["rb"], first)
                    first = NO_BASIS
                else:
                    run_steps(state, n_local, {"gtab": blk["gtab"], "steps": [st]})
        elif it["kind"] == 1:
            port.ims_swap(state.view(np.float64), n_local, [tuple(p) for p in it["pairs"]])
        else:
            raise AssertionError("cross-rank item")
    return state


def support_after(st, tmask, smask, sval):
    """Known-zero coset after a pass (schedule.h supportAfter): tile bits that
    no non-diagonal gate touched stay fixed, moved by the store permutation."""
    m, v = smask & ~tmask, sval & ~tmask
    for frm, to in st.get("keep", []):
        if (smask >> frm) & 1:
            m |= 1 << to
            v |= ((sval >> frm) & 1) << to
    return m, v


def run_program_jit_sparse(qk, port, prog, n_local, state, initial):
    """As the runtime runs a program from |basis> with known zeros: the first
    pass computes ONLY the tile holding |basis> (no memset: `state` may hold
    garbage, e.g. NaN), later passes get the known-zero coset (smask, sval)
    and skip what lies outside it.  Requires the program to start with a
    block of >= 2 passes (else the runtime zero-fills)."""
    os.environ["QK_DEBUG_FROM_BASIS"] = "1"  # the schedule qk_simulate runs (free initial layout)
    qk.set_jit_min_qubits(0)
    try:
        d = prog.debug_compile(n_local)
        srcs = iter(prog.debug_jit_sources(n_local))
    finally:
        qk.set_jit_min_qubits(22)
        del os.environ["QK_DEBUG_FROM_BASIS"]
    items = d["items"]
    basis = sum(((initial >> p) & 1) << m for p, m in enumerate(d["mem0"]))  # initial in the start layout
    full = (1 << n_local) - 1
    smask, sval, first = full, basis, True
    for it in items:
        if it["kind"] == 0:
            blk = it["block"]
            gt = np.array(blk["gtab"] if blk["gtab"] else [0.0, 0.0], dtype=np.float64)
            steps = blk["steps"]
            for si, st in enumerate(steps):
                if st["kind"] != 0:
                    run_steps(state, n_local, {"gtab": blk["gtab"], "steps": [st]})
                    for q in st["targets"]:
                        smask &= ~(1 << q)
                    continue
                name, src = next(srcs)
                tmask = sum(1 << b for b in st["tile_phys"])
                fn = host_kernel2(name, src)
                if first:  # only the basis tile: compacted non-tile bits of basis
                    t, q = 0, 0
                    for b in range(n_local):
                        if not (tmask >> b) & 1:
                            t |= ((basis >> b) & 1) << q
                            q += 1
                    fn(state.ctypes.data, gt.ctypes.data, n_local, st["ct"], st["rb"], basis, t, t + 1, 0, 0, 0)
                    first = False
                else:
                    # deferred zeros (as the runtime): a sparse pass followed by a pass,
                    # with the support still partial after it, leaves its zero tiles unwritten
                    nxt = si + 1 < len(steps) and steps[si + 1]["kind"] == 0
                    amask, _ = support_after(st, tmask, smask, sval)
                    defer = bool(smask and amask and nxt)
                    # deferred zeros launch only the tiles meeting the support (zskip 2)
                    tiles = 1 << (n_local - st["ct"] - bin(smask & ~tmask).count("1")) if defer else 0
                    fn(state.ctypes.data, gt.ctypes.data, n_local, st["ct"], st["rb"], NO_BASIS, 0, tiles, smask,
                       sval if smask else 0, 2 if defer else 0)
                smask, sval = support_after(st, tmask, smask, sval)
        elif it["kind"] == 1:
            pairs = [tuple(p) for p in it["pairs"]]
            port.ims_swap(state.view(np.float64), n_local, pairs)
            def sw(x):
                for o, i in pairs:
                    d = ((x >> o) ^ (x >> i)) & 1
                    x ^= (d << o) | (d << i)
                return x
            smask, sval = sw(smask), sw(sval)
        else:
            raise AssertionError("cross-rank item")
    return state
