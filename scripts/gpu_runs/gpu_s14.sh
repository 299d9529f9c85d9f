export PYTHONPATH=.
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_outer_parity.py -q -k "solvers_match or outer_loop" 2>&1 | tail -15
