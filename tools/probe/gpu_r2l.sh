O=gpurun_out/r2l; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2l
for k in qft bvones qaoa random grover; do
  timeout 300 python tools/family_passes.py $k 33 > $O/fam_$k.txt 2> $O/fam_$k.err; cat $O/fam_$k.txt | grep -v "^----"; sed -n '/---- tuned run/,$p' $O/fam_$k.err | grep "qk item" | tr '\n' ' ' | cut -c1-300; echo
done
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc $?"; cat $O/bench.json; tail -3 $O/bench.err
timeout 1700 python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -15 $O/pytest_gpu.log
