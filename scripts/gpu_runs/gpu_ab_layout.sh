export PYTHONPATH=.
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "hv" 2>&1 | tail -3
HV_IMPL=tc_f16 bash scripts/ab_lib.sh 3 lib_base.so lib_lay1.so lib_epi4.so lib_epi4lay1.so
timeout 300 python bench.py --no-outer --no-large --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['e2e']['value'])"
