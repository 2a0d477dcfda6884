#!/bin/bash
# One gpurun session: GPU tests, smoke, bench lines (HV, Wan), the ncu launch
# list of one bench step and full ncu captures of K3 / K1 / K2.
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [tag]'
set -u
TAG=${1:-r01}
O=gpurun_out/$TAG
mkdir -p "$O"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > "$O/gpu.txt" 2>&1
lscpu > "$O/lscpu.txt" 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$O/pytest_gpu.log"
timeout -s KILL 300 python __graft_entry__.py --smoke > "$O/smoke.log" 2>&1; echo "smoke rc=$?" >> "$O/smoke.log"
timeout -s KILL 900 python bench.py > "$O/bench_hv.log" 2>&1
timeout -s KILL 600 python bench.py --config wan --no-cpu-baseline > "$O/bench_wan.log" 2>&1
timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 1 > "$O/bench_ref.log" 2>&1
# launch list of one profiled bench step (cold-cache, serialised: compare shares)
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$O/launches.csv" python bench.py --profile --steps 2 --warmup 3 > "$O/ncu_launches.log" 2>&1
# full captures: K3 (one launch), K1, K2
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc_pair -s 3 -c 1 \
  -o "$O/k3" python bench.py --profile --steps 1 --warmup 3 > "$O/ncu_k3.log" 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"pool_warp|select_rows|dgemm|text_combine" -s 4 -c 4 \
  -o "$O/k12" python bench.py --profile --steps 1 --warmup 3 > "$O/ncu_k12.log" 2>&1
ls -la "$O"
for f in pytest_gpu smoke; do tail -n 2 "$O/$f.log"; done; for f in bench_hv bench_wan bench_ref; do tail -n 1 "$O/$f.log"; done
