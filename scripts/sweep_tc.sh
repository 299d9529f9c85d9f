#!/bin/bash
# Ablation sweep of the tcgen05 H.V at config 1 (env knobs of hv_tc.cu).
cd "$(dirname "$0")/.."
for impl in tc tc_bf16; do
T="timeout 60 python scripts/time_hv.py $impl 13500 26 65 50"
$T
WGP_TC_CHUNK=100000 $T
WGP_TC_DEBUG=17 $T
WGP_TC_DEBUG=23 WGP_TC_CHUNK=100000 $T
WGP_TC_TRACE=1 $T 2>&1 | tail -2
done
