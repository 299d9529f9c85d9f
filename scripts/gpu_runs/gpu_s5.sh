export PYTHONPATH=.
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/s5_launches.csv python scripts/time_hv.py tc_f16 13500 26 65 10 > /dev/null 2>&1
for i in tc_f16 tc; do HV_IMPL=$i timeout 300 python scripts/time_ap.py c3; done
