#!/bin/bash
# DP flop weight sweep (QK_DP_FLOP) on every family at 33 qubits.
O=gpurun_out/r2t; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2t
for f in 60 120 250; do for C in qft bvones qaoa random grover; do
  QK_DP_FLOP=$f timeout 900 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --circuit $C > $O/$C.flop$f.json 2> $O/$C.flop$f.err
  echo "$C flop$f rc=$?" >> $O/status.txt
done; done
