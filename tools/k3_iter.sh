#!/bin/bash
# K3 iteration: the d = B = 128 parity tests, then one HV bench line (no CPU leg).
#   gpurun --timeout 1200 -- 'bash tools/k3_iter.sh <tag> [extra bench args]'
set -u
TAG=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
timeout -s KILL 600 python -m pytest tests -m gpu -x -q -k "pair_pingpong or headline or tcgen05 or errors" > $O/pytest_k3.log 2>&1; echo "rc=$?" >> $O/pytest_k3.log
tail -3 $O/pytest_k3.log
timeout -s KILL 600 python bench.py --no-cpu-baseline --no-extras --steps 10 --warmup 3 "$@" > $O/bench.log 2>&1
tail -1 $O/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',round(d['value'],3), {k: round(x,3) for k,x in d['kernels_ms'].items()}, 'TF', round(d['roofline']['achieved'],1), d.get('clocks'))" || tail -20 $O/bench.log
