#!/bin/bash
# A/B builds in tools/ab_so/*.so on one box (RSA_B200_LIB selects the library):
#   tools/ab_lib.sh name1 name2 ...   (each run twice, interleaved)
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for v in "$@"; do
    printf "%-10s " "$v"
    RSA_B200_LIB=tools/ab_so/$v.so timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline \
      --no-extras --e2e-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), {k: round(x,3) for k,x in d['kernels_ms'].items()}, d['clocks']['sm_mhz'])" 2>&1 | tail -1
  done
done
