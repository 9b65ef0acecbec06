O=gpurun_out/r2c; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2c
timeout 600 python -m pytest tests/test_gpu_kernels.py -k u5 -m gpu -q -x > $O/pytest_u5.log 2>&1; echo "pytest u5 rc $?"; tail -15 $O/pytest_u5.log
timeout 600 python tools/u5bench.py 30 3 > $O/u5_30.txt 2>&1; echo "u5 30 rc $?"; cat $O/u5_30.txt
timeout 600 python tools/u5bench.py 33 2 > $O/u5_33.txt 2>&1; echo "u5 33 rc $?"; cat $O/u5_33.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_tile -c 2 -o $O/prof_u5 python tools/u5bench.py 28 1 > $O/ncu_u5.log 2>&1; echo "ncu rc $?"; tail -3 $O/ncu_u5.log
