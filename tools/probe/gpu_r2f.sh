O=gpurun_out/r2f; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2f
timeout 1500 python -m pytest tests -m gpu -q -x --durations=25 > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -45 $O/pytest_gpu.log
for k in qft bvones qaoa random grover; do
  timeout 300 python tools/family_passes.py $k 33 2>/dev/null | grep -v "^----" | sed "s/^/new: /"
  QK_ROW_PEN=1,0.6,0.3,0 QK_XCHG_COST=0 timeout 300 python tools/family_passes.py $k 33 2>/dev/null | grep -v "^----" | sed "s/^/old: /"
done
U5_MODES=0,1 timeout 600 python tools/u5bench.py 33 2
