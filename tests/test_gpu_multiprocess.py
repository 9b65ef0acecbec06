"""Multi-process runs: one process per rank, the N>1 path bench.py takes under
torchrun.  Each rank owns a slice; cross-rank swaps go over peer memory
(qk_ipc_init: cudaIpc-mapped slices + in-place swap kernel) -- which also runs
with several processes on this single-GPU box -- or over NCCL (qk_comm_init:
grouped ncclSend/ncclRecv + single receive buffer + copy-back), which needs
one GPU per rank and is skipped on a 1-GPU box.

Checked against the reference: spawnRanks (distributed.cpp:140-206) states
within 1e-10 plus the final layout, and xrsSwap (distributed.cpp:124-138)
bit-exact with its RankStats."""
import json
import os
import subprocess
import sys
import uuid

import numpy as np
import pytest

from conftest import ROOT
from oracle import config_text

pytestmark = pytest.mark.gpu
WORKER = os.path.join(ROOT, "tests", "mp_rank.py")


def gpus():
    import paper_2409_14697_b200 as qk
    return qk.device_count()


def launch(tmp_path, spec, ranks, transport="ipc"):
    job = f"t{uuid.uuid4().hex[:12]}"
    spec_path = tmp_path / f"{job}.json"
    spec_path.write_text(json.dumps(spec))
    procs = []
    env = dict(os.environ, QK_IPC_TIMEOUT="120")
    for r in range(ranks):
        procs.append(subprocess.Popen([sys.executable, WORKER, "--rank", str(r), "--job", str(tmp_path / job) if
                                       transport == "nccl" else job, "--spec", str(spec_path), "--out",
                                       str(tmp_path / f"{job}_{r}"), "--transport", transport], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
    outs = []
    for r, p in enumerate(procs):
        try:
            log, _ = p.communicate(timeout=300)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        assert p.returncode == 0, f"rank {r}: {log.decode()[-2000:]}"
    for r in range(ranks):
        outs.append((np.load(tmp_path / f"{job}_{r}.npy"), json.load(open(tmp_path / f"{job}_{r}.json"))))
    return outs


CASES = [  # (n, R, B, kind, a, seed, flags)
    (12, 1, 11, "qft", 0, 0, {}),
    (14, 2, 12, "random", 120, 5, dict(fusion=0, diag=0)),
    (15, 2, 6, "qaoa", 1, 3, {}),
    (13, 3, 10, "random", 80, 9, dict(c=6)),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_ipc_program_vs_spawnranks(ref, tmp_path, case):
    n, r, b, kind, a, seed, flags = CASES[case]
    flags = dict(flags)
    c = flags.pop("c", min(10, n - r))
    cfg_text = config_text(n, r, c, b=b, **flags)
    prog = ref.optimize(ref.gen(kind, n, a, seed), cfg_text)
    assert "CSQS" in prog
    initial = 0x2A5 & ((1 << n) - 1)
    want, wl, _, _ = ref.simulate(prog, cfg_text, n, r, initial, 0)
    spec = {"n": n, "r": r, "b": b, "mode": "program", "program": prog, "config": cfg_text, "initial": initial,
            "runs": 2}
    outs = launch(tmp_path, spec, 1 << r)
    got = np.concatenate([o[0] for o in outs])
    assert np.max(np.abs(got - want.view(np.complex128))) < 1e-10
    assert abs(np.sum(np.abs(got) ** 2) - 1.0) < 1e-12


@pytest.mark.parametrize("n,r,b,pairs", [(10, 1, 9, [(3, 9)]), (12, 2, 10, [(9, 10), (2, 11)]),
                                         (11, 3, 8, [(7, 8), (1, 9), (5, 10)]), (13, 2, 4, [(10, 12)])])
def test_ipc_xrs_swap_bitexact(ref, tmp_path, n, r, b, pairs):
    rng = np.random.default_rng(n * 7 + r)
    full = rng.standard_normal(2 << n)
    path = tmp_path / "state.npy"
    np.save(path, full)
    want = full.copy()
    wstats = ref.xrs_swap(want, n, r, b, pairs)
    spec = {"n": n, "r": r, "b": b, "mode": "xrs", "state": str(path), "pairs": pairs}
    outs = launch(tmp_path, spec, 1 << r)
    got = np.concatenate([o[0] for o in outs])
    assert np.array_equal(got.view(np.float64), want)
    for k, (_, meta) in enumerate(outs):
        assert tuple(meta["stats"]) == tuple(int(x) for x in wstats[k])


def test_ipc_large_slices(tmp_path):
    # 2 ranks x 2^27 amplitudes (2 GiB each) on this GPU: a QFT-28 with its
    # CSQS items over peer memory, against the closed form on sampled windows
    import paper_2409_14697_b200 as qk
    from test_gpu_programs import qft_expected
    n, r = 28, 1
    cfg = qk.Config.make(n, r, chunk=13, fusion=0, diag=0)
    prog = qk.Program.optimize(qk.generate("qft", n), cfg)
    assert prog.counts()["csqs"] > 0
    spec = {"n": n, "r": r, "b": cfg.buffer_qubits, "mode": "program", "program": prog.text(),
            "config": cfg.text(), "initial": 0x1234567, "runs": 1}
    outs = launch(tmp_path, spec, 2)
    got = np.concatenate([o[0] for o in outs])
    p2l = prog.final_layout()
    for off in (0, (1 << n) - (1 << 20), 3 << 25):
        want = qft_expected(n, 0x1234567, p2l, np.arange(off, off + (1 << 20), dtype=np.int64))
        assert np.max(np.abs(got[off:off + (1 << 20)] - want)) < 1e-10
    assert abs(np.sum(np.abs(got) ** 2) - 1.0) < 1e-12


def test_nccl_program_vs_spawnranks(ref, tmp_path):
    if gpus() < 2:
        pytest.skip("NCCL needs one GPU per rank (NCCL rejects two ranks on one device)")
    n, r, b = 14, 1, 10
    cfg_text = config_text(n, r, 10, b=b)
    prog = ref.optimize(ref.gen("qft", n), cfg_text)
    want, _, _, _ = ref.simulate(prog, cfg_text, n, r, 3, 0)
    spec = {"n": n, "r": r, "b": b, "mode": "program", "program": prog, "config": cfg_text, "initial": 3}
    outs = launch(tmp_path, spec, 2, transport="nccl")
    got = np.concatenate([o[0] for o in outs])
    assert np.max(np.abs(got - want.view(np.complex128))) < 1e-10
