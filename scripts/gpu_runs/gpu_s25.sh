export PYTHONPATH=.
for sp in 0 1 2 3 4 6; do echo "splits=$sp $(WGP_I8_SPLITS=$sp timeout 300 python scripts/time_cg64_c2.py | tr '\n' ' ')"; done
