#!/bin/bash
# Interleaved A/B timing of env-knob variants on one box (box-to-box variance
# is ~20%, so variants are only compared within one run).
# usage: ab.sh IMPL N REPS "ENV_A" "ENV_B" ...
cd "$(dirname "$0")/.."
impl=$1; n=$2; reps=$3; shift 3
for r in $(seq $reps); do
  for v in "$@"; do
    env $v timeout 60 python scripts/time_hv.py $impl $n 26 65 30 2>&1 | tail -1 | sed "s/^/[$v] /"
  done
done | sort | awk '{print}'
