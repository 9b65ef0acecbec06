O=gpurun_out/r2k; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2k
for k in bvones qft grover; do
  QK_DEBUG_TUNE=1 timeout 300 python tools/family_passes.py $k 33 > $O/fam_$k.txt 2> $O/fam_$k.err; cat $O/fam_$k.txt | grep -v "^----"
done
timeout 900 python -m pytest tests/test_gpu_programs.py tests/test_gpu_full_size.py tests/test_gpu_large_parity.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc $?"; tail -3 $O/pytest.log
timeout 600 python tools/ref_cpu_full.py 30 > $O/ref30.json 2>&1; cat $O/ref30.json
timeout 1500 python tools/ref_cpu_full.py 33 > $O/ref33.json 2>&1; cat $O/ref33.json
