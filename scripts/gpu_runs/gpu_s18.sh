export PYTHONPATH=.
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/s18.csv python scripts/time_cg64_c2.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hv_i8_kernel -s 3 -c 1 -o gpurun_out/s18_i8 python scripts/time_cg64_c2.py > /dev/null 2>&1
