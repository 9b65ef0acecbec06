"""Per-block device time of a program's blocks applied one by one
(qk.apply_block, each block its own pass): python tools/blockbench.py N [chunk] [kind]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_14697_b200 as qk
n = int(sys.argv[1]); chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 13
kind = sys.argv[3] if len(sys.argv) > 3 else "qft"
cfg = qk.Config.make(n, 0, chunk=chunk, fusion=0, diag=0)
prog = qk.Program.optimize(qk.generate(kind, n, {"qaoa": 1, "random": 400}.get(kind, 0), 7), cfg).text()
lines = prog.splitlines(); blocks = []; i = 0
while i < len(lines):
    k = int(lines[i])
    if not lines[i + 1].startswith(("SQS", "CSQS")):
        blocks.append(lines[i + 1:i + 1 + k])
    i += 1 + k
st = qk.State(n)
st.set_basis(0)
tag = os.environ.get("TAG", "")
tot = 0.0
for b in blocks:
    qk.apply_block(st, b, chunk); st.synchronize()  # compile + warm
    t0 = time.perf_counter(); qk.apply_block(st, b, chunk); st.synchronize(); dt = time.perf_counter() - t0
    tot += dt
    kinds = {}
    for g in b: kinds[g.split()[0]] = kinds.get(g.split()[0], 0) + 1
    print(f"{tag} {dt*1e3:8.2f} ms {32*(1<<n)/dt/1e9:7.0f} GB/s  {kinds}", flush=True)
print(f"{tag} total {tot*1e3:.1f} ms over {len(blocks)} blocks, avg {32*(1<<n)*len(blocks)/tot/1e9:.0f} GB/s")
