export PYTHONPATH=.
for r in 1 2; do for l in lib_e16g16 lib_e8g32 lib_e8g16; do
  echo "$l $(WGP_LIBRARY=$PWD/ab/$l.so timeout 300 python scripts/time_cg64_c2.py | tr '\n' ' ')"
done; done
