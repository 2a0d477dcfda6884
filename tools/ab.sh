#!/bin/bash
# A/B of K3 variants within one GPU session: bench.py K3 time per variant/mode
for v in "$@"; do
  echo "== $v"
  env $v timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), {k: round(x,3) for k,x in d['kernels_ms'].items()}, round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
