#!/bin/bash
# One GPU call: tests, bench line, ncu launch list, one full capture of the top kernel.
# Usage (under gpurun): bash tools/gpu_round.sh [tag]
TAG=${1:-r1}
O=gpurun_out/$TAG
mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache
nvidia-smi > $O/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?"; tail -3 $O/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc $?"; cat $O/bench.json; tail -3 $O/bench.err
if [ "${SKIP_NCU:-0}" = "0" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/bench_ncu.log 2>&1; echo "ncu-list rc $?"
# the two full-state passes of QFT-31 (launch 0 is the synthesized single-tile pass)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qk_pass -s 1 -c 2 -o $O/prof_block \
   python tools/run_qft.py 31 > $O/ncu_full.log 2>&1; echo "ncu-full rc $?"; tail -3 $O/ncu_full.log
fi
