#!/bin/bash
# gradient kernel ablations at config 3 (same box): WGP_GRAD_DEBUG bits
export PYTHONPATH=.
for dbg in 0 1 2 3 4 5; do
  echo "dbg=$dbg"; WGP_GRAD_DEBUG=$dbg timeout 120 python scripts/time_grad.py c3 2 2>&1 | grep " tc:"
done
