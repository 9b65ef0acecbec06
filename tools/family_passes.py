"""Per-pass device times of a circuit family after autotune (QK_PROFILE_ITEMS
prints one line per pass / IMS to stderr): python tools/family_passes.py KIND N"""
import os
import sys
os.environ["QK_PROFILE_ITEMS"] = "1"  # read once, at the first profiled run
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_14697_b200 as qk

kind = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 33
a, seed = {"qft": (0, 0), "bvones": (0, 0), "qaoa": (1, 1), "random": (400, 7), "grover": (1, 5)}[kind]
cfg = qk.Config.make(n, 0, chunk=13, fusion=0, diag=0)
prog = qk.Program.optimize(qk.generate(kind, n, a, seed), cfg)
st = qk.State(n)
for _ in range(24):
    if not st.simulate(prog, 0)["tuning_runs"]:
        break
st.set_profiling(True)
print("---- tuned run", flush=True)
sys.stderr.write("---- tuned run\n")
sys.stderr.flush()
s = st.simulate(prog, 0)
print(f"{kind}-{n}: total {s['total_ms']:.2f} ms, full passes {s['full_pass_launches']} in {s['full_pass_ms']:.2f} ms "
      f"({s['full_pass_bytes'] / (s['full_pass_ms'] * 1e-3) / 1e9 if s['full_pass_ms'] else 0:.0f} GB/s), "
      f"init {s['init_ms']:.2f} ms, ims {s['ims_ms']:.2f} ms", flush=True)
