#!/bin/bash
# PP kernel: repeated race checks (tcgen05 vs CUDA-core K3), then an A/B
export RSA_TC_PP=1
for i in $(seq 1 ${N:-8}); do timeout -s KILL 120 python tools/tc_vs_simt.py ${TT:-0} 2>&1 | tail -1; done
unset RSA_TC_PP
[ -n "$AB" ] && bash tools/ab.sh RSA_TC_PP=0 RSA_TC_PP=1 RSA_TC_PP=0 RSA_TC_PP=1
exit 0
