#!/bin/bash
# A/B of the support-aware DP pricing (QK_SPARSE_DP) on every family at 33 qubits.
mkdir -p gpurun_out/r2x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2x/gpu.txt
for c in qft bvones qaoa random grover; do
  for v in 0 1; do
    QK_SPARSE_DP=$v timeout 900 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --circuit $c > gpurun_out/r2x/$c.dp$v.json 2> gpurun_out/r2x/$c.dp$v.err
    echo "$c dp=$v rc=$?" >> gpurun_out/r2x/status.txt
  done
done
