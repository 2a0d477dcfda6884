#!/bin/bash
# per-step traces of one CTA for both K3 kernels
O=gpurun_out/$1; mkdir -p $O
for kv in 1 2; do
  for cta in 5000 9000; do
    echo "== RSA_TC_KERNEL=$kv cta=$cta"; RSA_TC_KERNEL=$kv RSA_TC_TRACE_CTA=$cta timeout 120 python tools/tc_trace.py 2>&1 | tail -45
  done
done > $O/trace.log 2>&1
cat $O/trace.log | grep -E "==|median"
