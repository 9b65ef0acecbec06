"""One rank of a multi-process run (tests/test_gpu_multiprocess.py launches
2^R of these): its slice on cuda:<device>, the rank group over peer memory
(qk_ipc_init) or NCCL (qk_comm_init), then either a whole program
(spawnRanks semantics, distributed.cpp:140-206) or one xrsSwap on uploaded
slices (distributed.cpp:124-138).  Writes its slice (and stats) to --out."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, required=True)
    ap.add_argument("--job", required=True)
    ap.add_argument("--spec", required=True)  # JSON: n, r, b, mode, program/config or state/pairs, initial
    ap.add_argument("--out", required=True)
    ap.add_argument("--transport", default="ipc", choices=["ipc", "nccl"])
    a = ap.parse_args()
    import paper_2409_14697_b200 as qk
    spec = json.load(open(a.spec))
    n, r, b = spec["n"], spec["r"], spec["b"]
    ranks = 1 << r
    device = a.rank % max(1, qk.device_count()) if a.transport == "nccl" else spec.get("device", 0)
    st = qk.State(n, r, a.rank, b, device)
    if a.transport == "ipc":
        st.ipc_init(a.job, ranks, a.rank)
    else:
        import time
        idf = a.job + ".ncclid"
        if a.rank == 0:
            with open(idf + ".tmp", "wb") as f:
                f.write(qk.comm_unique_id())
            os.replace(idf + ".tmp", idf)
        while not os.path.exists(idf):
            time.sleep(0.01)
        st.comm_init(open(idf, "rb").read(), ranks, a.rank)
    out = {}
    if spec["mode"] == "program":
        cfg = qk.Config.parse(spec["config"])
        prog = qk.Program.parse(spec["program"], cfg)
        for _ in range(spec.get("runs", 1)):
            stats = st.simulate(prog, spec["initial"])
        out["xrs_rounds"] = stats["xrs_rounds"]
    else:
        full = np.load(spec["state"]).view(np.complex128)
        sl = full[a.rank << (n - r):(a.rank + 1) << (n - r)]
        st.upload(sl)
        out["stats"] = list(st.xrs_swap([tuple(p) for p in spec["pairs"]]))
    np.save(a.out + ".npy", st.download())
    json.dump(out, open(a.out + ".json", "w"))
    st.close()


if __name__ == "__main__":
    main()
