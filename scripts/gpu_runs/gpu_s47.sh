export PYTHONPATH=.
for l in lib_full lib_nomma lib_nomath; do for s in 64 65; do
  echo "$l s=$s $(WGP_LIBRARY=$PWD/ab/$l.so timeout 300 python scripts/time_cg64_c2.py c2 $s 2>&1 | tr '\n' ' ')"
done; done
