"""Debug: run growing prefixes of a program on the GPU (interpreter and
specialized kernels) and compare each with the reference build's
run_items on the same prefix.  python tools/bisect_prefix.py N chunk [kind]"""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import paper_2409_14697_b200 as qk
from oracle import Ref, config_text
n = int(sys.argv[1]); chunk = int(sys.argv[2]); kind = sys.argv[3] if len(sys.argv) > 3 else "qft"
ref = Ref()
cfg_text = config_text(n, 0, chunk, fusion=0, diag=0)
prog = ref.optimize(ref.gen(kind, n, {"qaoa": 1, "random": 300}.get(kind, 0), 7), cfg_text)
lines = prog.splitlines(); items = []; i = 0
while i < len(lines):
    k = int(lines[i]); items.append(lines[i:i + 1 + k]); i += 1 + k
cfg = qk.Config.parse(cfg_text)
init = 12345
for k in range(1, len(items) + 1):
    if items[k - 1][1].startswith("SQS"):
        continue
    text = "\n".join(l for it in items[:k] for l in it) + "\n"
    want = np.zeros(2 << n); want[2 * init] = 1
    ref.run_items(text, cfg_text, want, 0, k, os.cpu_count())
    want = want.view(np.complex128)
    p = qk.Program.parse(text, cfg)
    errs = []
    for jit in (-1, 0):
        qk.set_jit_min_qubits(jit)
        st = qk.State(n); st.simulate(p, init)
        errs.append(float(np.max(np.abs(st.download() - want)))); st.close()
    print(f"prefix {k:3d} items  interp {errs[0]:.2e}  jit {errs[1]:.2e}  last block {len(items[k-1])-1} gates", flush=True)
    if max(errs) > 1e-10:
        print("FIRST BAD PREFIX", k); print("\n".join(items[k - 1][:40])); break
