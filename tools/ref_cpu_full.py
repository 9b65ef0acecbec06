"""One real reference run at full size on the host cores (no extrapolation):
the reference's simulateProgram (oracle/_ref, unmodified sources) on
QFT-N with the bench's program (chunk_qbit 13, fusion off), all host threads.
The state stays inside the reference (no copy-out), so QFT-33 needs 128 GiB of
host RAM.  python tools/ref_cpu_full.py N"""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import Ref, config_text  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 33
threads = os.cpu_count() or 1
ref = Ref()
cfg = config_text(n, 0, 13, fusion=0, diag=0)
prog = ref.optimize(ref.gen("qft", n), cfg)
p2l = (C.c_int * n)()
sec = C.c_double()
t0 = time.perf_counter()
rc = ref.lib.ref_simulate(prog.encode(), cfg.encode(), 0, threads, None, p2l, None, C.byref(sec))
wall = time.perf_counter() - t0
mem = open("/proc/meminfo").read().split("\n")[0]
print(json.dumps({"workload": f"QFT-{n} (chunk_qbit 13, fusion off)", "rc": rc, "threads": threads,
                  "simulate_s": round(sec.value, 3), "wall_s_incl_alloc": round(wall, 3), "host": mem}), flush=True)
