#!/bin/bash
# Quick GPU iteration: GPU tests for the specialized kernels + programs, then the bench line.
TAG=${1:-q}; O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_programs.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc $?"; tail -3 $O/pytest.log
timeout 900 python bench.py --no-cpu-baseline --steps 2 > $O/bench.json 2> $O/bench.err; echo "bench rc $?"
python - $O/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value",d["value"],"block",d["breakdown"]["block_ms"],"ims",d["breakdown"]["ims_ms"],"frac",d["roofline"]["frac"],"clk",d["clocks"]["sm_mhz"],d["clocks"]["reasons"])
PY
tail -3 $O/bench.err
