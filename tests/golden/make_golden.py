"""Regenerate the golden fixtures from the REFERENCE build (run in the builder
container, where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

Every vector here is an output of the unmodified reference (oracle/_ref/
libquokka_ref.so = /root/reference/proj/src compiled as-is), so the GPU tests
can pin parity on the GPU box where /root/reference does not exist.

  golden_programs.json  generator circuits + configs -> reference Program text
  golden_states.npz     reference simulateProgram / spawnRanks / applyBlock /
                        imsSwap / xrsSwap outputs on seeded inputs
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import Ref, config_text, random_state  # noqa: E402

SHOWCASE = ("H 0 0\nH 1 1\nRZZ 2 4 2 2\nRZZ 5 7 3 3\nH 8 4\nH 9 5\nH 3 6\nH 6 7\n"
            "RZZ 0 2 8 8\nRZZ 4 7 9 9\nH 9 10\nRZZ 1 8 11 11\nRZZ 3 6 12 12\nH 5 13\n")

# (name, generator kind, n, a, seed, config kwargs)
PROGRAM_CASES = [
    ("qft10_default", "qft", 10, 0, 0, dict(r=0)),
    ("qft12_c5_unfused", "qft", 12, 0, 0, dict(r=0, c=5, fusion=0, diag=0)),
    ("qft12_c6_fused", "qft", 12, 0, 0, dict(r=0, c=6, f=3)),
    ("qaoa9_p2", "qaoa", 9, 2, 11, dict(r=0, c=4)),
    ("bvones11_f5", "bvones", 11, 0, 0, dict(r=0, c=6, f=5)),
    ("random11_r2", "random", 11, 80, 7, dict(r=2, c=4)),
    ("random12_r1_b6", "random", 12, 120, 3, dict(r=1, c=5, b=6, fusion=0)),
    ("random10_r3", "random", 10, 60, 19, dict(r=3, c=4, diag=0)),
    ("qft11_r2_unfused", "qft", 11, 0, 0, dict(r=2, c=4, fusion=0, diag=0)),
    ("qaoa10_r1", "qaoa", 10, 1, 5, dict(r=1, c=5)),
]


def main():
    r = Ref()
    programs = {}
    arrays = {}
    # Showcase (proj/tests/fixtures.hpp:21-35) at the reference tests' config.
    for name, kw in (("showcase_plain", dict(fusion=0, diag=0)), ("showcase_fused", {})):
        cfg = config_text(10, 2, 4, **kw)
        prog = r.optimize(SHOWCASE, cfg)
        programs[name] = dict(circuit=SHOWCASE, config=cfg, program=prog, n=10, r=2)
    for name, kind, n, a, seed, kw in PROGRAM_CASES:
        circ = r.gen(kind, n, a, seed)
        cfg = config_text(n, **kw)
        prog = r.optimize(circ, cfg)
        programs[name] = dict(circuit=circ, config=cfg, program=prog, n=n, r=kw.get("r", 0))
    for name, case in programs.items():
        for initial in (0, 5):
            st, p2l, stats, _ = r.simulate(case["program"], case["config"], case["n"], case["r"], initial, 2)
            arrays[f"{name}/init{initial}/state"] = st
            arrays[f"{name}/init{initial}/phys_to_log"] = np.array(p2l, dtype=np.int32)
            if stats is not None:
                arrays[f"{name}/init{initial}/stats"] = stats.astype(np.uint64)

    # applyBlock on a seeded random state: every gate kind (test_engine.cpp:167-233 style).
    blocks = {
        "mixed": ["H 0 0", "X 2 1", "U 1 2 0.3 1.1 -0.7", "RX 3 3 0.9", "RY 0 4 -1.3", "RZ 2 5 2.2",
                  "RZZ 1 3 6 0.8", "CP 0 3 7 1.9", "CX 3 1 8", "CX 0 2 9", "SWAP 1 2 10", "CP 3 0 11 -0.6"],
    }
    for seed in range(3):
        circ = r.gen("random", 5, 24, 500 + seed)
        blocks[f"random5_{seed}"] = [ln for ln in circ.splitlines() if ln.strip()]
    for name, lines in blocks.items():
        n = 9
        chunk = 4 if name == "mixed" else 5
        st = random_state(n, 600 + len(name))
        arrays[f"block/{name}/in"] = st.copy()
        r.apply_block(st, n, lines, chunk, 1)
        arrays[f"block/{name}/out"] = st
        programs[f"block/{name}"] = dict(lines=lines, n=n, chunk=chunk)

    # imsSwap: random disjoint pair sets (test_engine.cpp:114-151 style).
    rng = np.random.default_rng(99)
    ims_cases = []
    for t in range(8):
        n = int(rng.integers(6, 13))
        qs = rng.permutation(n)
        s = int(rng.integers(1, n // 2 + 1))
        pairs = sorted((int(min(qs[2 * i], qs[2 * i + 1])), int(max(qs[2 * i], qs[2 * i + 1]))) for i in range(s))
        st = random_state(n, 1000 + t)
        arrays[f"ims/{t}/in"] = st.copy()
        r.ims_swap(st, n, pairs, int(rng.integers(0, 4)), 1)
        arrays[f"ims/{t}/out"] = st
        ims_cases.append(dict(n=n, pairs=pairs))
    programs["ims_cases"] = ims_cases

    # xrsSwap: a few (n, R, S, B) shapes (test_distributed.cpp:104-161 style).
    xrs_cases = []
    for t, (n, R, S, B) in enumerate([(6, 2, 2, 2), (8, 2, 1, 6), (9, 3, 3, 4), (10, 3, 2, 7), (7, 1, 1, 1)]):
        region = n - R
        outs = sorted(int(x) for x in rng.choice(region, S, replace=False))
        ins = sorted(int(x) for x in rng.choice(np.arange(region, n), S, replace=False))
        pairs = list(zip(outs, ins))
        st = random_state(n, 2000 + t)
        arrays[f"xrs/{t}/in"] = st.copy()
        stats = r.xrs_swap(st, n, R, B, pairs)
        arrays[f"xrs/{t}/out"] = st
        arrays[f"xrs/{t}/stats"] = stats.astype(np.uint64)
        xrs_cases.append(dict(n=n, r=R, s=S, b=B, pairs=pairs))
    programs["xrs_cases"] = xrs_cases

    with open(os.path.join(HERE, "golden_programs.json"), "w") as f:
        json.dump(programs, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "golden_states.npz"), **arrays)
    print("wrote", len(programs), "program cases,", len(arrays), "arrays")


if __name__ == "__main__":
    main()
