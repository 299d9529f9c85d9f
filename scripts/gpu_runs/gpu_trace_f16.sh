export PYTHONPATH=.
L=$PWD/ab/lib_ablate.so
echo "== trace"; WGP_LIBRARY=$L WGP_TC_TRACE=1 timeout 120 python scripts/time_hv.py tc_f16 13500 26 65 5 2>&1 | tail -8
echo "== trace tc"; WGP_LIBRARY=$L WGP_TC_TRACE=1 timeout 120 python scripts/time_hv.py tc 13500 26 65 5 2>&1 | tail -8
for r in 1 2; do
for dbg in 0 1 2 4 8 16 32 128 512 6 ; do
  echo "dbg=$dbg $(WGP_LIBRARY=$L WGP_TC_DEBUG=$dbg timeout 60 python scripts/time_hv.py tc_f16 13500 26 65 30 2>&1 | tail -1)"
done
echo "default $(timeout 60 python scripts/time_hv.py tc_f16 13500 26 65 30 2>&1 | tail -1)"
done
