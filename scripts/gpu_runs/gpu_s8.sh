export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
HV_IMPL=tc_f16 bash scripts/ab_lib.sh 3 lib_base.so lib_new.so
HV_IMPL=tc bash scripts/ab_lib.sh 2 lib_base.so lib_new.so
