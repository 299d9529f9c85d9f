#!/bin/bash
# config-0 CG outer loop, A/B of library builds on one box: ab_c0.sh REPS lib_a.so lib_b.so ...
cd "$(dirname "$0")/.."
export PYTHONPATH=.
reps=$1; shift
for r in $(seq $reps); do
  for lib in "$@"; do
    WGP_LIBRARY=$PWD/ab/$lib timeout 120 python scripts/c0_steps.py 2>&1 | tail -1 | sed "s/^/[$lib] /"
  done
done | sort
