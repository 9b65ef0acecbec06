export QK_JIT_CACHE=$PWD/gpurun_out/jitcache
timeout 900 python tools/bisect_prefix.py 24 13 > gpurun_out/bisect24.log 2>&1; tail -50 gpurun_out/bisect24.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1; tail -15 gpurun_out/pytest_all.log
