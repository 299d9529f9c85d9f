#!/bin/bash
# A/B of (library build, env) variants on one box: ab_lib_env.sh REPS "lib_a.so ENV=.." "lib_b.so" ...
cd "$(dirname "$0")/.."
export PYTHONPATH=.
reps=$1; shift
for r in $(seq $reps); do
  for v in "$@"; do
    set -- $v
    lib=$1; shift
    env WGP_LIBRARY=$PWD/ab/$lib "$@" timeout 60 python scripts/time_hv.py ${HV_IMPL:-tc_f16} 13500 26 65 30 2>&1 | tail -1 | sed "s/^/[$v] /"
  done
done | sort
