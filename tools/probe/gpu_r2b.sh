O=gpurun_out/r2b; mkdir -p $O
export QK_JIT_CACHE=/tmp/qk_jit_cache_r2b
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -m gpu -q -x --durations=10 > $O/pytest_mp.log 2>&1; echo "pytest mp rc $?"; tail -30 $O/pytest_mp.log
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc $?"; cat $O/bench.json; tail -5 $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 2 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc $?"; cat $O/bench_ref.json; tail -3 $O/bench_ref.err
timeout 900 python -m pytest tests/test_gpu_jit.py -m gpu -q -x --durations=5 > $O/pytest_jit.log 2>&1; echo "pytest jit rc $?"; tail -8 $O/pytest_jit.log
