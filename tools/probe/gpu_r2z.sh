#!/bin/bash
# Deferred H scales A/B, GPU suite, bench line + reference arm, launch list, QFT-31 ncu, family per-pass times.
O=gpurun_out/r2z; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2z
for C in qft bvones qaoa; do for v in 0 1; do
  QK_DEFER_H=$v timeout 900 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --circuit $C > $O/$C.defer$v.json 2> $O/$C.defer$v.err
  echo "$C defer=$v rc=$?" >> $O/status.txt
done; done
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status.txt
timeout 1200 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/status.txt
for k in qft bvones qaoa random grover; do
  timeout 600 python tools/family_passes.py $k 33 > $O/fam_$k.txt 2> $O/fam_$k.err
done
echo "fam done" >> $O/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_ncu.log 2>&1; echo "ncu-list rc $?" >> $O/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qk_pass -s 1 -c 2 -o $O/prof_qft31 python tools/run_qft.py 31 > $O/ncu_qft.log 2>&1; echo "ncu qft rc $?" >> $O/status.txt
QK_TUNE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:qk_pass -c 20 -o /tmp/prof_grover31 -f python tools/run_qft.py 31 13 1 grover > $O/ncu_grover.log 2>&1; echo "ncu grover rc $?" >> $O/status.txt
python tools/ncu_summary.py /tmp/prof_grover31.ncu-rep --sass > $O/summary_grover.txt 2>&1
