export PYTHONPATH=.
for r in 1 2; do for l in lib_cur lib_f2dalu2; do
  echo "$l $(WGP_LIBRARY=$PWD/ab/$l.so timeout 300 python scripts/time_cg64_c2.py | tr '\n' ' ')"
done; done
