O=gpurun_out/r2g; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2g
timeout 1700 python -m pytest tests -m gpu -q --durations=30 > $O/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -50 $O/pytest_gpu.log
