#!/bin/bash
# GPU parity tests + bench lines: bash tools/run_bench.sh <tag> [extra bench args...]
set -u
TAG=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log
timeout -s KILL 900 python bench.py --no-cpu-baseline "$@" > $O/bench.log 2>&1
tail -1 $O/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',round(d['value'],3), {k: round(x,3) for k,x in d['kernels_ms'].items()}, 'e2e', d['e2e'] and round(d['e2e']['value'],2), 'TF', round(d['roofline']['achieved'],1), d.get('clocks'))" || tail -20 $O/bench.log
