#!/bin/bash
# gradient kernel cluster size (R_J multicast) A/B at config 3 and 2, same box
export PYTHONPATH=.
for cs in 1 2 4 2 1; do
  echo "cs=$cs"; WGP_GRAD_CLUSTER=$cs timeout 120 python scripts/time_grad.py c3 2 2>&1 | grep " tc:"
done
for cs in 1 2 4; do
  echo "cs=$cs"; WGP_GRAD_CLUSTER=$cs timeout 120 python scripts/time_grad.py c2 3 2>&1 | grep " tc:"
done
