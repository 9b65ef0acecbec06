"""Time the fused-U5 tile kernel, DFMA vs DMMA, on BV-n with fusion_qbit 5
(every U5 of the reference-default fused program): python tools/u5bench.py N [reps]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_14697_b200 as qk

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = qk.Config.make(n, 0, chunk=13, fusion_qubits=5)
prog = qk.Program.optimize(qk.generate("bvones", n), cfg)
u5 = prog.text().count("U5 ")
st = qk.State(n)
st.set_profiling(True)
modes = [int(m) for m in os.environ.get("U5_MODES", "2,0,1").split(",")]
for mode, name in [(m, {0: "DFMA", 1: "DMMA", 2: "generic k_dense_group"}[m]) for m in modes]:
    qk.set_dense_mode(mode)
    ts = []
    for _ in range(reps):
        s = st.simulate(prog, 0)
        ts.append(s["block_ms"] - s["full_pass_ms"] - s["init_ms"])
    dense_ms = min(ts)
    per = dense_ms / u5
    flops = 256.0 * (1 << n)  # 32x32 complex matvec per 32 amps: 8*32 real flops per amp
    print(f"{name}: {u5} U5 gates, {dense_ms:.2f} ms total, {per:.3f} ms per U5, "
          f"{flops / (per * 1e-3) / 1e12:.2f} TFLOP/s, {32.0 * (1 << n) / (per * 1e-3) / 1e9:.0f} GB/s; "
          f"total step {s['total_ms']:.1f} ms", flush=True)
qk.set_dense_mode(-1)
