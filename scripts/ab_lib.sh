#!/bin/bash
# Interleaved A/B of two library builds (ab/lib_*.so) on one box: config-1
# H.V kernel time.  usage: ab_lib.sh REPS lib_a.so lib_b.so ...
cd "$(dirname "$0")/.."
export PYTHONPATH=.
reps=$1; shift
for r in $(seq $reps); do
  for lib in "$@"; do
    WGP_LIBRARY=$PWD/ab/$lib timeout 60 python scripts/time_hv.py ${HV_IMPL:-tc_f16} 13500 26 65 30 2>&1 | tail -1 | sed "s/^/[$lib] /"
  done
done | sort
