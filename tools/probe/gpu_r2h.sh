O=gpurun_out/r2h; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2h
for k in qft bvones qaoa random grover; do
  timeout 300 python tools/family_passes.py $k 33 2>/dev/null | grep -v "^----"
done
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc $?"; cat $O/bench.json; tail -3 $O/bench.err
timeout 1700 python -m pytest tests -m gpu -q --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -25 $O/pytest_gpu.log
