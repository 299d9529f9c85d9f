export PYTHONPATH=.
for r in 1 2; do for l in lib_g8 lib_g16; do
  echo "$l $(WGP_LIBRARY=$PWD/ab/$l.so timeout 300 python scripts/time_cg64_c2.py | tr '\n' ' ')"
done; done
WGP_LIBRARY=$PWD/ab/lib_g16.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "engines or i8" 2>&1 | tail -2
