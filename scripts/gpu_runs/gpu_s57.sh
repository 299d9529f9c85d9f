export PYTHONPATH=.
timeout 300 python scripts/time_cg64_c2.py
timeout 300 ncu --metrics gpu__time_duration.sum -k regex:i8_vimg -c 2 --csv python scripts/time_hv64_kernel.py 65 2>/dev/null | grep i8_vimg | awk -F'","' '{print $NF}'
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "f64 or engines" 2>&1 | tail -2
