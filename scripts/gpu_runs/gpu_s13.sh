export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_outer_parity.py -x -q 2>&1 | tail -2
for i in tc_f16 tc; do HV_IMPL=$i timeout 300 python scripts/time_ap.py c3; done
HV_IMPL=tc_f16 timeout 300 python scripts/time_hv.py tc_f16 13500 26 65 30
