export PYTHONPATH=.
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 8000 --csv --log-file gpurun_out/s12_c3.csv python scripts/c3_step_profile.py > gpurun_out/s12_c3.out 2>&1
HV_IMPL=tc_f16 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 8000 --csv --log-file gpurun_out/s12_c3f16.csv python scripts/c3_step_profile.py > gpurun_out/s12_c3f16.out 2>&1
