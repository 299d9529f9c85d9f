export PYTHONPATH=.
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_outer_parity.py -x -q -k "f64 or cg or trajectory or solvers or outer" 2>&1 | tail -2
for r in 1 2; do
echo "x1 $(timeout 120 python scripts/time_cg64_c2.py 2>&1 | tail -2 | tr '\n' ' ')"
echo "nox1 $(WGP_HV64_NO_X1=1 timeout 120 python scripts/time_cg64_c2.py 2>&1 | tail -2 | tr '\n' ' ')"
done
timeout 300 python scripts/time_solvers.py 2>&1 | head -1
WGP_HV64_NO_X1=1 timeout 300 python scripts/time_solvers.py 2>&1 | head -1
