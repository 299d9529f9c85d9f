export PYTHONPATH=.
for r in 1 2; do for l in lib_t2 lib_t2nbk3; do
  echo "$l $(WGP_LIBRARY=$PWD/ab/$l.so timeout 300 python scripts/time_cg64_c2.py | tr '\n' ' ')"
done; done
