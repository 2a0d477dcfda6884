#!/bin/bash
# per-kernel device times of one profiled bench step under the given env: bash tools/launch_times.sh <tag> "<ENV=..>"...
O=gpurun_out/$1; shift; mkdir -p $O
i=0
for e in "$@"; do
  i=$((i+1))
  env $e timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/lt$i.csv \
    python bench.py --profile --steps 1 --warmup 2 > /dev/null 2>&1
  echo "== $e"
  python - $O/lt$i.csv <<'PY'
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
data = [(r[ki], float(r[vi].replace(',', ''))) for r in rows[hi + 1:] if len(r) > vi]
rsa = [(k, v) for k, v in data if 'rsa::' in k]
n = len(rsa) // 4   # warmup 2 + timed 1 + per-stage >=... take the last step's launches
last = collections.OrderedDict()
for k, v in rsa[-8:]:
    name = k.split('(')[0].replace('void rsa::<unnamed>::', '').replace('rsa::<unnamed>::', '')[:60]
    print(f"   {name:60s} {v/1e3:9.1f} us")
PY
done
