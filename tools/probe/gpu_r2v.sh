#!/bin/bash
# CTA-bit controls validation + knob A/B: GPU suite, families (new defaults, QK_CTA_CONTROLS=0),
# DP flop weight and persistent-prefetch A/B.
O=gpurun_out/r2v; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2v
run() { local C=$1 name=$2; shift 2
  env "$@" timeout 900 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --circuit $C > $O/$C.$name.json 2> $O/$C.$name.err
  echo "$C $name rc=$?" >> $O/status.txt; }
for C in qft bvones qaoa random grover; do run $C new QK_NOP=1; done
for C in random grover bvones; do run $C nocta QK_CTA_CONTROLS=0; done
run qft flop10 QK_DP_FLOP=10
run qft flop60 QK_DP_FLOP=60
run grover persist QK_JIT_PERSIST=1
run random persist QK_JIT_PERSIST=1
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
