#!/bin/bash
# A/B builds in tools/ab_so/*.so, REPS alternating rounds (default 4), K3 event times only:
#   REPS=4 tools/ab_lib_n.sh name1 name2 ...
cd "$(dirname "$0")/.."
for rep in $(seq 1 ${REPS:-4}); do
  for v in "$@"; do
    printf "%-8s " "$v"
    RSA_B200_LIB=tools/ab_so/$v.so timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline \
      --no-extras --e2e-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['kernels_ms']['attention'],3), d['clocks']['sm_mhz'])" 2>&1 | tail -1
  done
done
