#!/bin/bash
# Multi-rank bench path on one B200 at HEAD (all ranks on cuda:0, peer-memory XRS).
O=gpurun_out/r2mr2; mkdir -p $O
for N in 2 4; do
  QK_BENCH_SHARE_GPU=1 timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29$((500+N)) bench.py --gpus $N --per-gpu-qubits 28 --steps 5 --warmup 3 --no-cpu-baseline > $O/n$N.json 2> $O/n$N.err
  echo "N=$N rc=$?" >> $O/status.txt
done
