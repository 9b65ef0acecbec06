"""Multi-process (one process per rank) path on CPU: world_size 2 and 4 over
torch.distributed `gloo`, standing in for NCCL.

Each rank owns its 2^(N-R) slice (distributed.cpp:9-11) and executes exactly
the host plan the NCCL path executes (runtime.cpp runXrsNccl): the message
list from qk_xrs_plan (one grouped send/recv per partner per window round,
into one receive buffer section, then copy-back into the slab via
qk_xrs_slab_index).  Blocks run through the numpy replay of the compiled
pass programs (tests/emulator.py) and IMS through the oracle, so the whole
spawnRanks program (distributed.cpp:140-206) is checked against the reference
build with no GPU.  The XRS permutation itself is bit-exact
(test_distributed.cpp:104-161 semantics); programs are within 1e-10."""
import os
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT
from oracle import config_text, random_state


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _xrs_over_gloo(qk, sl, n, R, B, rank, pairs):
    """Execute this rank's XRS message list on its slice (in place)."""
    msgs = qk.xrs_plan(n, R, B, rank, pairs)
    outs = [p[0] for p in pairs]
    idx_cache = {}

    def idx(slab, w0, count):
        key = (slab, w0, count)
        if key not in idx_cache:
            idx_cache[key] = np.array([qk.xrs_slab_index(n, R, outs, slab, w0 + e) for e in range(count)],
                                      dtype=np.int64)
        return idx_cache[key]

    buf_amps = 0
    i = 0
    while i < len(msgs):
        j = i
        while j < len(msgs) and msgs[j]["round"] == msgs[i]["round"]:
            j += 1
        group = msgs[i:j]
        recv = {}
        reqs = []
        for m in group:
            send = torch.from_numpy(np.ascontiguousarray(sl[idx(m["slab"], m["w0"], m["count"])]).view(np.float64))
            rbuf = torch.empty(2 * m["count"], dtype=torch.float64)
            recv[m["section"]] = (m, rbuf)
            reqs.append(dist.isend(send, m["peer"]))
            reqs.append(dist.irecv(rbuf, m["peer"]))
            buf_amps = max(buf_amps, (m["section"] + 1) * m["count"])
        for r in reqs:
            r.wait()
        for sec, (m, rbuf) in recv.items():  # copy-back kernel
            sl[idx(m["slab"], m["w0"], m["count"])] = rbuf.numpy().view(np.complex128)
        i = j
    assert buf_amps <= (1 << B)  # single receive buffer of at most 2^B amplitudes
    return len({m["round"] for m in msgs})


def _worker(rank, world, port, task, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import paper_2409_14697_b200 as qk
    from emulator import run_steps
    from oracle import Port
    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    try:
        R = world.bit_length() - 1
        if task["kind"] == "xrs":
            n, B, pairs = task["n"], task["b"], [tuple(p) for p in task["pairs"]]
            full = np.load(task["state"])
            loc = 1 << (n - R)
            sl = full[rank * loc:(rank + 1) * loc].copy()
            rounds = _xrs_over_gloo(qk, sl, n, R, B, rank, pairs)
            np.save(os.path.join(outdir, f"r{rank}.npy"), sl)
            np.save(os.path.join(outdir, f"rounds{rank}.npy"), np.array([rounds]))
        else:
            n, initial = task["n"], task["initial"]
            cfg = qk.Config.parse(task["config"])
            prog = qk.Program.parse(task["program"], cfg)
            loc = 1 << (n - R)
            sl = np.zeros(loc, dtype=np.complex128)
            if initial >> (n - R) == rank:
                sl[initial & (loc - 1)] = 1
            port = Port()
            for it in prog.debug_compile(n - R)["items"]:
                if it["kind"] == 0:
                    run_steps(sl, n - R, it["block"])
                elif it["kind"] == 1:
                    port.ims_swap(sl.view(np.float64), n - R, [tuple(p) for p in it["pairs"]])
                else:
                    _xrs_over_gloo(qk, sl, n, R, cfg.buffer_qubits, rank, [tuple(p) for p in it["pairs"]])
            np.save(os.path.join(outdir, f"r{rank}.npy"), sl)
    finally:
        dist.destroy_process_group()


def _run(world, task):
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(world, _free_port(), task, d), nprocs=world, join=True,
                           start_method="spawn")
        out = np.concatenate([np.load(os.path.join(d, f"r{r}.npy")) for r in range(world)])
        rounds = [int(np.load(os.path.join(d, f"rounds{r}.npy"))[0]) for r in range(world)
                  if os.path.exists(os.path.join(d, f"rounds{r}.npy"))]
        return out, rounds


@pytest.mark.parametrize("world,n,b,pairs", [
    (2, 8, 7, [(6, 7)]),              # AIO-staged out (top in-rank position): contiguous slabs
    (2, 8, 3, [(1, 7)]),              # low out, windowed (B=3 -> several rounds)
    (4, 9, 7, [(5, 7), (6, 8)]),      # S=2 staged
    (4, 9, 4, [(0, 8), (3, 7)]),      # S=2 arbitrary outs, windowed
    (4, 9, 7, [(2, 8)]),              # S=1 of R=2: two independent groups
])
def test_xrs_over_gloo_bitexact(ref, world, n, b, pairs):
    st = random_state(n, 100 + n + b).view(np.complex128)
    with tempfile.NamedTemporaryFile(suffix=".npy", delete=False) as f:
        np.save(f, st)
    try:
        got, rounds = _run(world, {"kind": "xrs", "n": n, "b": b, "pairs": pairs, "state": f.name})
    finally:
        os.unlink(f.name)
    want = st.view(np.float64).copy()
    R = world.bit_length() - 1
    stats = ref.xrs_swap(want, n, R, b, pairs)
    assert np.array_equal(got.view(np.float64), want)
    assert rounds == [int(s[3]) for s in stats]  # reference's window-round count per rank


@pytest.mark.parametrize("world,kind,a,seed", [(2, "qft", 0, 0), (4, "random", 90, 5), (2, "qaoa", 1, 3)])
def test_program_over_gloo_vs_spawn_ranks(ref, world, kind, a, seed):
    n = 10
    R = world.bit_length() - 1
    cfg_text = config_text(n, R, 5, b=n - R - 1, fusion=0, diag=0)
    prog = ref.optimize(ref.gen(kind, n, a, seed), cfg_text)
    assert "CSQS" in prog
    want, _, _, _ = ref.simulate(prog, cfg_text, n, R, 7, 1)
    got, _ = _run(world, {"kind": "program", "n": n, "initial": 7, "config": cfg_text, "program": prog})
    assert np.max(np.abs(got - want.view(np.complex128))) < 1e-10
