#!/bin/bash
# BASELINE configs[2..3]: Wan bench line + sparsity sweep at the HV shape,
# IPAR+GAPR on (sparse-rectified) vs off (sparse-unrectified) vs the dense
# `full` variant of the same kernel.  bash tools/sweep.sh <tag>
O=gpurun_out/$1; mkdir -p $O; : > $O/sweep.jsonl
run() { timeout -s KILL 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 1 "$@" 2>&1 | tail -1 >> $O/sweep.jsonl; }
run --config wan
for s in 0.5 0.75 0.9 0.95; do
  for v in sparse-rectified sparse-unrectified; do run --sparsity $s --variant $v; done
done
run --variant full --steps 3
python - "$O/sweep.jsonl" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    try: d = json.loads(l)
    except Exception: print("ERR", l[:200]); continue
    c = d["config"]
    print(f'{c["workload"][:22]:22s} f={c["top_k_fraction"]:<5} {c["variant"]:20s} ms={d["value"]:8.3f} '
          f'K1={d["kernels_ms"]["pool"]:.3f} K2={d["kernels_ms"]["select"]:.3f} K3={d["kernels_ms"]["attention"]:.3f} '
          f'K3TF={d["roofline"]["achieved"]:.0f} sparsity={d["realized_sparsity"]:.4f} e2e={d["e2e"]["value"]:.1f}')
PY
