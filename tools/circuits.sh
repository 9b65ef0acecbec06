#!/bin/bash
# Bench line per circuit family (1 GPU): QFT-30, QFT-33, Grover-33, QAOA-33, random-33, BV-33.
O=gpurun_out/circ; mkdir -p $O
for args in "--circuit qft --per-gpu-qubits 30" "--circuit qft" "--circuit grover" "--circuit qaoa" "--circuit random" "--circuit bvones"; do
  timeout 900 python bench.py $args --steps 2 --warmup 3 > $O/out.json 2> $O/err.txt
  python - "$args" <<'PY'
import json,sys
try:
    d=json.loads(open('gpurun_out/circ/out.json').read().strip().splitlines()[-1]); b=d["breakdown"]
    print(f'{sys.argv[1]:36s} {d["config"]["workload"][:40]:40s} value {d["value"]:.4f} s  e2e {d["e2e"]["value"]:.4f}  block {b["block_ms"]:.0f} ({b["block_launches"]})  ims {b["ims_ms"]:.0f} ({b["ims_launches"]})  frac {d["roofline"]["frac"]}  prog_frac {b["program_roofline_frac"]}  cpu {d.get("cpu_baseline",{}).get("value")}')
except Exception as e:
    print(sys.argv[1], "FAILED", open('gpurun_out/circ/err.txt').read()[-400:])
PY
done
