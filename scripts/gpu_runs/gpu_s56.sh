export PYTHONPATH=.
for r in 1 2; do
echo "pdl   $(timeout 300 python scripts/time_cg64_c2.py | tr '\n' ' ')"
echo "nopdl $(WGP_I8_NO_PDL=1 timeout 300 python scripts/time_cg64_c2.py | tr '\n' ' ')"
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_outer_parity.py -q -x -k "f64 or engines or outer" 2>&1 | tail -2
