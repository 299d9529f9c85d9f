#!/bin/bash
# Interleaved timing of library variants: ab_libs.sh REPS IMPL "lib_a.so [ENV=..]" "lib_b.so" ...
cd "$(dirname "$0")/../.."
reps=$1; impl=$2; shift 2
for r in $(seq $reps); do
  for v in "$@"; do
    set -- $v
    lib=$1; shift
    env WGP_LIBRARY=$PWD/ab/$lib "$@" timeout 60 python scripts/diag_f16_time.py $impl ${SHAPE:-} 2>&1 | tail -1 | sed "s/^/[$v] /"
  done
done | sort
