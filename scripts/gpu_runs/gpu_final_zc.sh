export PYTHONPATH=.
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "zero_copy or row_chunks" 2>&1 | tail -5
timeout 300 python scripts/time_e2e_upload.py tc_f16 2>&1 | tail -12
timeout 300 python scripts/time_e2e_upload.py tc 4 2>&1 | tail -3
