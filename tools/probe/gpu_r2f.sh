#!/bin/bash
# Final round-2 batch at HEAD: GPU suite, bench line + reference arm, family lines,
# per-pass times, launch list, QFT-31 ncu.
O=gpurun_out/r2f; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2f
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status.txt
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/status.txt
timeout 1200 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/status.txt
for C in bvones qaoa random grover; do
  timeout 900 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --circuit $C > $O/$C.json 2> $O/$C.err; echo "$C rc=$?" >> $O/status.txt
done
timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 --per-gpu-qubits 30 > $O/qft30.json 2> $O/qft30.err; echo "qft30 rc=$?" >> $O/status.txt
for k in qft bvones qaoa random grover; do
  timeout 600 python tools/family_passes.py $k 33 > $O/fam_$k.txt 2> $O/fam_$k.err
done
echo "fam done" >> $O/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_ncu.log 2>&1; echo "ncu-list rc $?" >> $O/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qk_pass -s 1 -c 3 -o $O/prof_qft31 python tools/run_qft.py 31 > $O/ncu_qft.log 2>&1; echo "ncu qft rc $?" >> $O/status.txt
QK_TUNE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:qk_pass -c 20 -o /tmp/prof_grover31 -f python tools/run_qft.py 31 13 1 grover > $O/ncu_grover.log 2>&1; echo "ncu grover rc $?" >> $O/status.txt
python tools/ncu_summary.py /tmp/prof_grover31.ncu-rep --sass > $O/summary_grover.txt 2>&1
