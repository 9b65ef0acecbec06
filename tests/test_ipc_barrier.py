"""Host side of the peer-memory rank group (qk_ipc_init): the node-local
shared-memory rendezvous and barrier that bracket every cross-rank swap, run
by several processes on the CPU (no GPU needed)."""
import multiprocessing as mp
import os
import time
import uuid

import pytest


def _rank(job, n, r, rounds, q, timeout=30.0, delay=0.0):
    import paper_2409_14697_b200 as qk
    time.sleep(delay)
    t0 = time.perf_counter()
    try:
        qk.debug_host_barrier(job, n, r, rounds, timeout)
        q.put((r, "ok", time.perf_counter() - t0))
    except qk.SimulationError as e:
        q.put((r, str(e), time.perf_counter() - t0))


@pytest.mark.parametrize("n", [2, 4, 8])
def test_barrier_all_ranks_pass(n):
    job = f"cpu{uuid.uuid4().hex[:10]}"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_rank, args=(job, n, r, 200, q)) for r in range(n)]
    for p in ps:
        p.start()
    res = [q.get(timeout=60) for _ in range(n)]
    for p in ps:
        p.join(10)
    assert sorted(r for r, _, _ in res) == list(range(n))
    assert all(msg == "ok" for _, msg, _ in res), res
    assert not os.path.exists(f"/dev/shm/qk_{job}")  # rank 0 removes the name


def test_barrier_waits_for_a_late_rank():
    job = f"cpu{uuid.uuid4().hex[:10]}"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_rank, args=(job, 2, r, 3, q, 30.0, 1.5 if r == 1 else 0.0)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict((r, (m, t)) for r, m, t in (q.get(timeout=60) for _ in range(2)))
    for p in ps:
        p.join(10)
    assert res[0][0] == "ok" and res[1][0] == "ok"
    assert res[0][1] > 1.0  # rank 0 really waited for rank 1


def test_barrier_times_out_without_the_others():
    job = f"cpu{uuid.uuid4().hex[:10]}"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_rank, args=(job, 3, 0, 1, q, 1.0))
    p.start()
    r, msg, t = q.get(timeout=60)
    p.join(10)
    assert "timed out" in msg and t < 10
