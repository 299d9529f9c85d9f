export PYTHONPATH=.
L=$PWD/ab/lib_ablate.so
for r in 1 2; do for dbg in 0 2 4 6 8 32; do
  echo "dbg=$dbg $(WGP_LIBRARY=$L WGP_TC_DEBUG=$dbg timeout 60 python scripts/time_hv.py tc_f16 13500 26 65 30 2>&1 | tail -1)"
done; done
