#!/bin/bash
# H.V accuracy (dense config-3-like case) per library build: ab_lib_acc.sh lib_a.so ...
cd "$(dirname "$0")/.."
export PYTHONPATH=.
for lib in "$@"; do
  echo "[$lib] $(WGP_LIBRARY=$PWD/ab/$lib timeout 200 python scripts/diag_chunk_accuracy.py 32 2>&1 | tail -1)"
done
