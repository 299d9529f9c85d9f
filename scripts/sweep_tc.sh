#!/bin/bash
# Ablation sweep of the tcgen05 H.V at config 1 (env knobs of hv_tc.cu).
# dbg bits: 1 no epilogue math, 2 no MMA-2, 4 no MMA-1, 8 no V loads, 16 no
# epilogue TMEM traffic, 32 no B loads.
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv,noheader
for impl in tc tc_bf16; do
  for dbg in 0 1 17 23 63 6 40; do
    WGP_TC_CHUNK=100000 WGP_TC_DEBUG=$dbg timeout 60 python scripts/time_hv.py $impl 13500 26 65 50
  done
done
