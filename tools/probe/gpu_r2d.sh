O=gpurun_out/r2d; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2d
timeout 600 python -m pytest tests/test_gpu_kernels.py -k u5 -m gpu -q -x > $O/pytest_u5.log 2>&1; echo "pytest u5 rc $?"; tail -5 $O/pytest_u5.log
U5_MODES=2,0,1 timeout 600 python tools/u5bench.py 30 3 > $O/u5_30.txt 2>&1; echo "u5 30 rc $?"; cat $O/u5_30.txt
U5_MODES=0,1 timeout 600 python tools/u5bench.py 33 2 > $O/u5_33.txt 2>&1; echo "u5 33 rc $?"; cat $O/u5_33.txt
U5_MODES=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_tile -c 1 -o $O/prof_u5_mma python tools/u5bench.py 28 1 > $O/ncu_u5.log 2>&1; echo "ncu rc $?"; tail -2 $O/ncu_u5.log
U5_MODES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_tile -c 1 -o $O/prof_u5_fma python tools/u5bench.py 28 1 > $O/ncu_u5f.log 2>&1; echo "ncu rc $?"; tail -2 $O/ncu_u5f.log
