"""Time IMS kernels on the pair sets of the QFT-N materialization: python tools/imsbench.py N"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_14697_b200 as qk
n = int(sys.argv[1])
cfg = qk.Config.make(n, 0, chunk=13, fusion=0, diag=0)
p = qk.Program.optimize(qk.generate("qft", n), cfg)
sets = [it["pairs"] for it in p.debug_compile()["items"] if it["kind"] == 1]
sets += [[(0, n - 1)], [(0, n - 1), (1, n - 2), (2, n - 3)], [(5, n - 1), (6, n - 2)]]
st = qk.State(n)
st.set_basis(0)
tag = os.environ.get("QK_IMS_TILED", "2")
for pairs in sets:
    qk.ims_swap(st, pairs); st.synchronize()
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter(); qk.ims_swap(st, pairs); st.synchronize(); best = min(best, time.perf_counter() - t0)
    moved = 1 - 2.0 ** -len(pairs)
    print(f"mode {tag} S={len(pairs):2d} {best*1e3:8.2f} ms {32*(1<<n)*moved/best/1e9:7.0f} GB/s  {pairs[:4]}")
