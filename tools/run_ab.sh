#!/bin/bash
# GPU parity tests + A/B of K3 variants + one ncu capture: bash tools/run_ab.sh <tag> <env>...
set -u
TAG=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
bash tools/ab.sh "$@" > $O/ab.log 2>&1
cat $O/ab.log
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 3 -c 1 -o $O/k3 python bench.py --profile --steps 1 --warmup 3 > $O/ncu_k3.log 2>&1
tail -2 $O/ncu_k3.log
