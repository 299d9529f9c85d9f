export PYTHONPATH=.
mkdir -p gpurun_out
for i in 1 2; do
for cut in 0 8960 9216 8704 9472; do
  echo "cut=$cut"; WGP_HVDEV_CUT=$cut timeout 120 python scripts/time_hv.py tc_f16 2>&1 | tail -1
done; done > gpurun_out/ab_devcut.log 2>&1
for cut in 0 8960; do
  echo "cut=$cut"; WGP_HVDEV_CUT=$cut timeout 120 python scripts/time_hv.py tc 2>&1 | tail -1
done >> gpurun_out/ab_devcut.log 2>&1
cat gpurun_out/ab_devcut.log
S=$(date +%s)
( timeout 1500 python bench.py 2> gpurun_out/final_bench.err | tail -1 ) > gpurun_out/final_bench.json
echo "bench wall $(( $(date +%s) - S )) s"
cut -c1-700 gpurun_out/final_bench.json
