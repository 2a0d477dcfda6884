#!/bin/bash
# compute-sanitizer memcheck / synccheck / racecheck over tools/sanitize.py:
#   gpurun --timeout 2400 -- 'bash tools/sanitize.sh <tag>'
O=gpurun_out/$1; mkdir -p $O
for tool in memcheck synccheck racecheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    python tools/sanitize.py > $O/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 $O/sanitizer_$tool.log
done
