"""Time near-empty block passes (memory structure of the fused kernel) vs IMS."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_14697_b200 as qk
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
st = qk.State(n)
def t(fn, reps=5):
    fn(); best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); best = min(best, time.perf_counter() - t0)
    return best
for name, lines, chunk in [("rz0", ["RZ 0 0 0.1"], 13), ("rz12", ["RZ 12 0 0.1"], 13), ("h0", ["H 0 0"], 13),
                           ("h12", ["H 12 0"], 13), ("5h", [f"H {q} {q}" for q in range(8, 13)], 13),
                           ("13h", [f"H {q} {q}" for q in range(13)], 13)]:
    dt = t(lambda: qk.apply_block(st, lines, chunk))
    print(f"{name:6s} {dt*1e3:7.2f} ms {32*(1<<n)/dt/1e9:7.0f} GB/s")
dt = t(lambda: qk.ims_swap(st, [(20, 25)]))
print(f"ims hi  {dt*1e3:7.2f} ms {32*(1<<n)*0.5/dt/1e9:7.0f} GB/s (moved half)")
dt = t(lambda: qk.ims_swap(st, [(13, 20), (14, 21), (15, 22), (16, 23), (17, 24), (18, 25)]))
print(f"ims 6   {dt*1e3:7.2f} ms {32*(1<<n)*(1-2**-6)/dt/1e9:7.0f} GB/s")
