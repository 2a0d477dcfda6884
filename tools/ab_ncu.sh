#!/bin/bash
# A/B of library builds (tools/ab_so/<name>.so) by the K3 kernel's ncu duration:
# each launch runs alone at the unlocked clock, which makes sub-percent
# differences visible that the power-capped bench events hide.
#   REPS=2 tools/ab_ncu.sh name1 name2 ...
cd "$(dirname "$0")/.."
for rep in $(seq 1 ${REPS:-2}); do
  for v in "$@"; do
    printf "%-8s " "$v"
    RSA_B200_LIB=tools/ab_so/$v.so timeout -s KILL 200 ncu --metrics gpu__time_duration.sum --clock-control none \
      -k regex:"attn_tc_pair" -c 1 -s 2 python bench.py --profile --steps 1 --warmup 2 --no-cpu-baseline 2>&1 \
      | grep duration | awk '{print $NF}'
  done
done
