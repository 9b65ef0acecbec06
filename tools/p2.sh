O=gpurun_out/p2; mkdir -p $O
python tools/run_qft.py 30 13 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qk_pass -s 0 -c 2 -o $O/prof_tma python tools/run_qft.py 30 13 1 > $O/ncu.log 2>&1; echo "ncu rc $?"
timeout 900 python -m pytest tests/test_gpu_programs.py tests/test_gpu_kernels.py -m gpu -q --durations=12 > $O/dur.log 2>&1; tail -16 $O/dur.log
