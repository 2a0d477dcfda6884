#!/bin/bash
O=gpurun_out/$1; mkdir -p $O
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"pool_bulk|select_rows|dgemm" -s 4 -c 4 \
  -o $O/k12 python bench.py --profile --steps 1 --warmup 3 > $O/ncu_k12.log 2>&1
tail -2 $O/ncu_k12.log
