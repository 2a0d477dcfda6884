#!/bin/bash
# A/B two builds of librsa_b200.so on the same box: tools/ab_so/{base,new}.so, alternating
L=paper_2511_19835_b200/librsa_b200.so
cp $L /tmp/cur.so
for v in ${AB_ORDER:-base new base new}; do
  cp tools/ab_so/$v.so $L
  echo "== $v"
  timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 "$@" 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],3), {k: round(x,3) for k,x in d['kernels_ms'].items()}, d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
cp /tmp/cur.so $L
