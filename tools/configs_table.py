"""Device time of the BASELINE.json single-GPU configs (after autotune):
QFT-30 in the bench form (chunk 13, fusion off) and the reference-default
fused form (chunk 10, fusion 5, diagonal fusion), Grover-33, QFT-33, BV-33
(bench form and reference-default fusion).  python tools/configs_table.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_14697_b200 as qk

cases = [("QFT-30 bench form", "qft", 30, (0, 0), dict(chunk=13, fusion=0, diag=0)),
         ("QFT-30 reference defaults", "qft", 30, (0, 0), {}),
         ("QFT-33 bench form", "qft", 33, (0, 0), dict(chunk=13, fusion=0, diag=0)),
         ("Grover-33 bench form", "grover", 33, (1, 5), dict(chunk=13, fusion=0, diag=0)),
         ("BV-33 bench form", "bvones", 33, (0, 0), dict(chunk=13, fusion=0, diag=0)),
         ("BV-33 fusion_qbit 5", "bvones", 33, (0, 0), dict(chunk=13, fusion_qubits=5))]
for name, kind, n, (a, seed), kw in cases:
    cfg = qk.Config.make(n, 0, **kw)
    prog = qk.Program.optimize(qk.generate(kind, n, a, seed), cfg)
    st = qk.State(n)
    for _ in range(24):
        if not st.simulate(prog, 0)["tuning_runs"]:
            break
    ts = sorted(st.simulate(prog, 0)["total_ms"] for _ in range(5))
    st.close()
    print(f"{name:28s} {prog.counts()}  median {ts[2]:9.2f} ms", flush=True)
