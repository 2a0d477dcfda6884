#!/bin/bash
# PP correctness/perf session: logs under gpurun_out/pp/
O=gpurun_out/pp; mkdir -p $O
RSA_TC_PP=1 timeout -s KILL 600 python -m pytest tests -q -m gpu -x > $O/pytest_pp1.log 2>&1; tail -2 $O/pytest_pp1.log
timeout -s KILL 600 python -m pytest tests -q -m gpu -x > $O/pytest_pp0.log 2>&1; tail -2 $O/pytest_pp0.log
for v in 0 1 0 1 0 1; do
  RSA_TC_PP=$v timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench_$v.log 2>&1
  echo "PP=$v rc=$? $(tail -1 $O/bench_$v.log | cut -c1-60) $(python -c "import json; d=json.loads(open('$O/bench_$v.log').read().strip().splitlines()[-1]); print(d['kernels_ms']['attention'], d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
done
for i in $(seq 1 ${N:-6}); do RSA_TC_PP=1 timeout -s KILL 120 python tools/tc_vs_simt.py 0 2>&1 | tail -1; RSA_TC_PP=1 timeout -s KILL 120 python tools/tc_vs_simt.py 200 2>&1 | tail -1; done | sort | uniq -c
