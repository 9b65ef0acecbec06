O=gpurun_out/r2j; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2j
for k in qft bvones qaoa random grover; do
  QK_DEBUG_TUNE=1 timeout 300 python tools/family_passes.py $k 33 > $O/fam_$k.txt 2> $O/fam_$k.err; cat $O/fam_$k.txt | grep -v "^----"; grep "variant 3" $O/fam_$k.err | head -8 | tr '\n' ' '; echo
done
timeout 1500 python -m pytest tests/test_gpu_programs.py tests/test_gpu_full_size.py tests/test_gpu_large_parity.py tests/test_gpu_jit.py tests/test_gpu_multiprocess.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc $?"; tail -5 $O/pytest.log
