#!/bin/bash
# Exchange cost in the DP (QK_XCHG_COST) A/B on the families with many-segment passes.
O=gpurun_out/r2xc; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2xc
for v in 0.05 0.15; do for C in grover random qaoa qft; do
  QK_XCHG_COST=$v timeout 900 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --circuit $C > $O/$C.x$v.json 2> $O/$C.x$v.err
  echo "$C x$v rc=$?" >> $O/status.txt
done; done
