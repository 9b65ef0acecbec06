#!/bin/bash
# ncu captures of the QFT-30 program's passes (the top kernels) + launch list.
TAG=${1:-p}; O=gpurun_out/$TAG; mkdir -p $O
N=${N:-30}
python tools/run_qft.py $N 13 1 > /dev/null 2>&1   # warm the JIT cache
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qk_pass -s ${SKIP:-0} -c ${COUNT:-3} -o $O/prof_block \
   python tools/run_qft.py $N 13 1 > $O/ncu_full.log 2>&1; echo "ncu-full rc $?"; tail -2 $O/ncu_full.log
timeout 600 ncu --set full --clock-control none -k regex:k_ims -s 0 -c 2 -o $O/prof_ims \
   python tools/run_qft.py $N 13 1 > $O/ncu_ims.log 2>&1; echo "ncu-ims rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $O/launches.csv python tools/run_qft.py $N 13 2 > $O/launch.log 2>&1; echo "launches rc $?"
