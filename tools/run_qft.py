"""Run one QFT program on cuda:0 (for ncu captures): python tools/run_qft.py N [chunk] [reps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_14697_b200 as qk
n = int(sys.argv[1]); chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 13
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
kind = sys.argv[4] if len(sys.argv) > 4 else "qft"
cfg = qk.Config.make(n, 0, chunk=chunk, fusion=0, diag=0)
prog = qk.Program.optimize(qk.generate(kind, n, *{"qaoa": (1, 1), "random": (400, 7), "grover": (1, 5)}.get(kind, (0, 0))), cfg)
st = qk.State(n)
st.set_profiling(bool(os.environ.get("QK_PROFILE_ITEMS")))
for _ in range(reps):
    s = st.simulate(prog, 0)
print(prog.counts(), s["total_ms"], st.norm())
