#!/bin/bash
# A/B of bench.py runs given as "ENV=.. -- args" pairs separated by ';;'
#   bash tools/ab_args.sh "RSA_SELECT_REG=0 -- --weight-threshold 0.5" "RSA_SELECT_REG=1 -- --weight-threshold 0.5"
for spec in "$@"; do
  envs=${spec%%--*}; args=${spec#*--}
  echo "== $spec"
  env $envs timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 $args 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), {k: round(x,3) for k,x in d['kernels_ms'].items()}, d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
