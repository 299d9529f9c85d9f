export PYTHONPATH=.
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "cg or trajectory or paths" 2>&1 | tail -5
timeout 300 python scripts/time_solvers.py 2>&1 | head -2
WGP_CG_NO_FOLD=1 timeout 300 python scripts/time_solvers.py 2>&1 | head -2
timeout 600 python -m pytest tests/test_gpu_library_sharded.py tests/test_gpu_local_sharded.py -x -q 2>&1 | tail -3
