# bench + profiles after the int8-slice fp64 operator (run from the repo root under gpurun)
export PYTHONPATH=.
timeout 900 python bench.py > gpurun_out/s29_bench.json 2> gpurun_out/s29_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hv_i8_kernel -s 3 -c 1 -o gpurun_out/s29_hv_i8 python scripts/time_cg64_c2.py > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/s29_cg64_launches.csv python scripts/time_cg64_c2.py > /dev/null 2>&1
