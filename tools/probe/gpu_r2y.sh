#!/bin/bash
# Support-aware DP + tight support + Toffoli fusion: family benches (new defaults
# and each knob off), then the full GPU suite.
mkdir -p gpurun_out/r2y
run() { # name env...
  local name=$1; shift
  env "$@" timeout 900 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --circuit ${C} > gpurun_out/r2y/$C.$name.json 2> gpurun_out/r2y/$C.$name.err
  echo "$C $name rc=$?" >> gpurun_out/r2y/status.txt
}
for C in qft bvones qaoa random grover; do run new QK_NOP=1; done
C=grover; run noccx QK_FUSE_CCX=0
C=qaoa; run notight QK_TIGHT_SUPPORT=0
C=bvones; run notight QK_TIGHT_SUPPORT=0
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2y/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2y/status.txt
