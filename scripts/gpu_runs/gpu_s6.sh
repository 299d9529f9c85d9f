export PYTHONPATH=.
timeout 300 python scripts/time_solvers.py
HV_IMPL=tc_f16 timeout 300 python scripts/time_solvers.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/s6_c0.csv python scripts/c0_cg_launches.py > /dev/null 2>&1
