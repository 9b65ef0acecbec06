#!/bin/bash
# 16-B-row penalty for partial sparse passes (QK_SPARSE_PEN0 0 vs 8), smoke.
O=gpurun_out/r2r; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2r
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
for v in 0 8; do
  QK_SPARSE_PEN0=$v timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 --per-gpu-qubits 30 > $O/qft30.pen$v.json 2> $O/qft30.pen$v.err
  echo "qft30 pen$v rc=$?" >> $O/status.txt
  for C in qft bvones qaoa random grover; do
    QK_SPARSE_PEN0=$v timeout 900 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --circuit $C > $O/$C.pen$v.json 2> $O/$C.pen$v.err
    echo "$C pen$v rc=$?" >> $O/status.txt
  done
done
QK_PROFILE_ITEMS=1 timeout 300 python tools/family_passes.py qft 30 > $O/fam_qft30.txt 2> $O/fam_qft30.err
QK_SPARSE_PEN0=0 QK_PROFILE_ITEMS=1 timeout 300 python tools/family_passes.py qft 30 > $O/fam_qft30_pen0.txt 2> $O/fam_qft30_pen0.err
