export PYTHONPATH=.
for r in 1 2; do for l in lib_i8e8 lib_i8e16; do
  echo "$l $(WGP_LIBRARY=$PWD/ab/$l.so timeout 300 python scripts/time_cg64_c2.py | tr '\n' ' ')"
done; done
WGP_LIBRARY=$PWD/ab/lib_i8e16.so timeout 300 python scripts/diag_i8.py gpurun_out/e16.npz 2>&1 | tail -4
