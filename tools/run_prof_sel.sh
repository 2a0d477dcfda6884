#!/bin/bash
O=gpurun_out/$1; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"select_rows|pool_bulk" -s 2 -c 2 \
  -o $O/sel python bench.py --profile --steps 1 --warmup 2 > $O/ncu_sel.log 2>&1
tail -1 $O/ncu_sel.log
