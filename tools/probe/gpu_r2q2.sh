#!/bin/bash
O=gpurun_out/r2q2; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2q2
for v in 0 8; do
  QK_SPARSE_PEN0=$v timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 --per-gpu-qubits 30 > $O/qft30.pen$v.json 2> $O/qft30.pen$v.err
  for C in random qft; do
    QK_SPARSE_PEN0=$v timeout 900 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --circuit $C > $O/$C.pen$v.json 2> $O/$C.pen$v.err
  done
  echo "pen$v done" >> $O/status.txt
done
