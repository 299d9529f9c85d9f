export PYTHONPATH=.
L=$PWD/ab/lib_ablate.so
echo "== trace f16 (4 groups, A_I in smem)"; WGP_LIBRARY=$L WGP_TC_TRACE=1 timeout 120 python scripts/time_hv.py tc_f16 13500 26 65 5 2>&1 | tail -8
for dbg in 0 1 16; do
  echo "dbg=$dbg $(WGP_LIBRARY=$L WGP_TC_DEBUG=$dbg timeout 60 python scripts/time_hv.py tc_f16 13500 26 65 30 2>&1 | tail -1)"
done
for sp in 3 4 5 6 8; do echo "splits=$sp $(WGP_TC_SPLITS=$sp timeout 60 python scripts/time_hv.py tc_f16 13500 26 65 30 2>&1 | tail -1)"; done
