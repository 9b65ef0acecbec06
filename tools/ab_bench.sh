#!/bin/bash
# A/B of tuning knobs on the bench line (no CPU baseline).  Usage: bash tools/ab_bench.sh "ENV=.. ENV2=.." ...
for cfg in "$@"; do
  env $cfg timeout 600 python bench.py --no-cpu-baseline --steps 2 --warmup 3 ${BENCH_ARGS} > /tmp/ab.json 2>/tmp/ab.err
  python - "$cfg" <<'PY'
import json,sys
try:
    d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1])
    b=d["breakdown"]
    print(f'{sys.argv[1]:40s} value {d["value"]:.4f}  block {b["block_ms"]:.1f} ({b["block_launches"]})  ims {b["ims_ms"]:.1f} ({b["ims_launches"]})  clk {d["clocks"]["sm_mhz"]} {d["clocks"]["reasons"]}')
except Exception as e:
    print(sys.argv[1], "FAILED", open('/tmp/ab.err').read()[-300:])
PY
done
