# round-2 session-3 bench + profiles (run from the repo root under gpurun)
export PYTHONPATH=.
timeout 900 python bench.py > gpurun_out/s9_bench.json 2> gpurun_out/s9_bench.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s9_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-outer --no-large > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hv_tc_kernel -s 5 -c 1 -o gpurun_out/s9_hv_tc_f16 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-outer --no-large > /dev/null 2>&1
timeout 300 python bench.py --impl reference > gpurun_out/s9_ref.json 2> gpurun_out/s9_ref.err
