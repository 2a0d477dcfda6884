#!/bin/bash
# K1 occupancy variants (tools/ab_so/k1_<ctas>_<stages>.so): K1 time per variant, alternating
L=paper_2511_19835_b200/librsa_b200.so
cp $L /tmp/cur.so
for rep in 1 2 3; do for v in k1_3_2 k1_5_1 k1_4_1; do
  cp tools/ab_so/$v.so $L
  echo "$v $(timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['kernels_ms']['pool'],3))")"
done; done
cp /tmp/cur.so $L
