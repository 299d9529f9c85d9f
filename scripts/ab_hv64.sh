#!/bin/bash
# A/B of hv_f64 kernel builds (ab/lib_*.so): ncu kernel durations at configs 0, 1, 2.
cd "$(dirname "$0")/.."
export PYTHONPATH=.
for lib in "$@"; do
  for c in "c0 17" "c1 65" "c2 65"; do
    t=$(WGP_LIBRARY=$PWD/ab/$lib ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"hv64p?_kernel" --csv \
        python scripts/time_hv64.py $c 3 2>/dev/null | grep -E "hv64p?_kernel" | tail -1 | awk -F'","' '{print $NF}' | tr -d '"')
    echo "[$lib] $c hv64_kernel ns=$t"
  done
done
