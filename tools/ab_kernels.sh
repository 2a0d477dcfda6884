#!/bin/bash
# A/B of K3 kernels by name on one box: bash tools/ab_kernels.sh kern1 kern2 ... (each twice, interleaved)
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for v in "$@"; do
    printf "%-20s " "$v"
    timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --e2e-steps 0 --kernel $v 2>&1 | \
      tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), {k: round(x,3) for k,x in d['kernels_ms'].items()}, d['clocks']['sm_mhz'])" 2>&1 | tail -1
  done
done
