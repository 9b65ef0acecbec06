"""Compare the GPU kernel against the numpy emulator op by op (debug aid)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]
import numpy as np
import paper_2409_14697_b200 as qk
from emulator import run_steps
cases = {
    "H0": ["H 0 0"], "H5": ["H 5 0"], "X2": ["X 2 0"], "X2H2": ["X 2 0", "H 2 1"],
    "U1": ["U 1 2 0.3 1.1 -0.7"], "RZ2": ["RZ 2 0 0.7"], "RZ7": ["RZ 7 0 0.7"],
    "CP01": ["CP 0 1 0 0.9"], "CP07": ["CP 0 7 0 0.9"], "CP78": ["CP 7 8 0 0.9"],
    "RZZ13": ["RZZ 1 3 0 0.8"], "RZZ17": ["RZZ 1 7 0 0.8"], "RZZ78": ["RZZ 7 8 0 0.8"],
    "CX31": ["CX 3 1 0"], "CX71": ["CX 7 1 0"], "X3CX31": ["X 3 0", "CX 3 1 1"],
    "SWAP12": ["SWAP 1 2 0"], "X2SWAP12H1": ["X 2 0", "SWAP 1 2 1", "H 1 2"],
    "mixedA": ["H 0 0", "X 2 1", "U 1 2 0.3 1.1 -0.7", "RX 3 3 0.9", "RY 0 4 -1.3", "RZ 2 5 2.2"],
    "mixedB": ["RZZ 1 3 6 0.8", "CP 0 3 7 1.9", "CX 3 1 8", "CX 0 2 9", "SWAP 1 2 10", "CP 3 0 11 -0.6"],
}
n = 9
rng = np.random.default_rng(0)
for name, lines in cases.items():
    st = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    want = st.copy()
    run_steps(want, n, qk.debug_compile_block(lines, n))
    d = qk.State(n); d.upload(st); qk.apply_block(d, lines, n); got = d.download()
    print(f"{name:12s} {np.max(np.abs(got - want)):.3e}")
