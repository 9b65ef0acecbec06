O=gpurun_out/r2e; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2e
timeout 600 python -m pytest tests/test_gpu_kernels.py -k u5 -m gpu -q -x > $O/pytest_u5.log 2>&1; echo "pytest u5 rc $?"; tail -3 $O/pytest_u5.log
U5_MODES=0,1 timeout 600 python tools/u5bench.py 33 2 > $O/u5_33.txt 2>&1; echo "u5 33 rc $?"; cat $O/u5_33.txt
U5_MODES=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_tile -c 1 -o $O/prof_u5_mma python tools/u5bench.py 28 1 > $O/ncu_u5.log 2>&1; echo "ncu rc $?"
U5_MODES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dense_tile -c 1 -o $O/prof_u5_fma python tools/u5bench.py 28 1 > $O/ncu_u5f.log 2>&1; echo "ncu rc $?"
for k in qft bvones grover qaoa random; do
  QK_DEBUG_TUNE=1 timeout 600 python tools/family_passes.py $k 33 > $O/fam_$k.txt 2> $O/fam_$k.err; echo "fam $k rc $?"; cat $O/fam_$k.txt; sed -n '/---- tuned run/,$p' $O/fam_$k.err | head -40
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qk_pass -s 1 -c 3 -o $O/prof_bv python tools/run_qft.py 31 13 1 bvones > $O/ncu_bv.log 2>&1; echo "ncu bv rc $?"
