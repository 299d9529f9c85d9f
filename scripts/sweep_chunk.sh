#!/bin/bash
# Time vs accumulation chunk (tiles) for both tensor-core precisions at config 1.
cd "$(dirname "$0")/.."
for impl in tc tc_bf16; do
  for ch in 4 8 16 32 100000; do
    WGP_TC_CHUNK=$ch timeout 60 python scripts/time_hv.py $impl 13500 26 65 50
  done
done
