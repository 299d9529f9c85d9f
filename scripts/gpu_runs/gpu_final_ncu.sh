export PYTHONPATH=.
mkdir -p gpurun_out
timeout 600 python bench.py --no-outer --no-large --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/final_b.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --no-outer --no-large --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/final_ncu.log 2>&1
tail -2 gpurun_out/final_ncu.log | cut -c1-300
wc -l gpurun_out/final_launches.csv
( timeout 1500 python bench.py 2> gpurun_out/final_bench2.err | tail -1 ) > gpurun_out/final_bench2.json
tail -1 gpurun_out/final_bench2.err
