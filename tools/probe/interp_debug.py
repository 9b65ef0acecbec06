import sys, os
sys.path[:0] = [os.getcwd(), os.path.join(os.getcwd(), "oracle")]
import numpy as np
import paper_2409_14697_b200 as qk
from oracle import Ref, config_text
ref = Ref()
qk.set_jit_min_qubits(-1)
for kind, a in (("qft", 0), ("random", 150), ("qaoa", 1)):
    for n in (12, 13, 14, 16, 18, 20, 22, 24):
        cfg_text = config_text(n, 0, min(13, n), fusion=0, diag=0)
        pt = ref.optimize(ref.gen(kind, n, a, 3), cfg_text)
        want = ref.simulate(pt, cfg_text, n, 0, 5, 8)[0].view(np.complex128)
        prog = qk.Program.parse(pt, qk.Config.parse(cfg_text))
        for initial_path in ("synth",):
            st = qk.State(n)
            st.simulate(prog, 5)
            got = st.download()
            st.close()
            d = prog.debug_compile(n)
            cts = sorted({s['ct'] for it in d['items'] if it['kind'] == 0 for s in it['block']['steps'] if s['kind'] == 0})
            print(kind, n, "cts", cts, "err %.3e" % np.max(np.abs(got - want)), flush=True)
