export PYTHONPATH=.
for r in 1 2 3; do
echo "pdl   $(TIME_HV_NOPROF=1 timeout 60 python scripts/time_hv.py tc_f16 13500 26 65 30 | tail -1)"
echo "nopdl $(WGP_TC_NO_PDL=1 TIME_HV_NOPROF=1 timeout 60 python scripts/time_hv.py tc_f16 13500 26 65 30 | tail -1)"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "hv or solvers" 2>&1 | tail -2
