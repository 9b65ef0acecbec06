"""Per-item device timing of a program: python tools/profile_items.py N [chunk] [kind]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_14697_b200 as qk
n = int(sys.argv[1]); chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 13
kind = sys.argv[3] if len(sys.argv) > 3 else "qft"
cfg = qk.Config.make(n, 0, chunk=chunk, fusion=0, diag=0)
prog = qk.Program.optimize(qk.generate(kind, n, {"qaoa": 1, "random": 400}.get(kind, 0), 7), cfg).text()
st = qk.State(n)
lines = prog.splitlines(); i = 0; items = []
while i < len(lines):
    k = int(lines[i]); items.append(lines[i + 1:i + 1 + k]); i += 1 + k
for rep in range(2):
    tot = 0
    for body in items:
        t0 = time.perf_counter()
        if body[0].startswith("SQS"):
            t = body[0].split(); s = int(t[1])
            qk.ims_swap(st, list(zip(map(int, t[2:2 + s]), map(int, t[2 + s:]))))
            what = body[0][:60]
        else:
            qk.apply_block(st, body, chunk)
            kinds = {}
            for b in body: kinds[b.split()[0]] = kinds.get(b.split()[0], 0) + 1
            what = f"block {kinds}"
        dt = time.perf_counter() - t0; tot += dt
        if rep == 1:
            print(f"{dt*1e3:8.2f} ms {32*(1<<n)/dt/1e9:7.0f} GB/s  {what}")
    if rep == 1: print("total", tot)
