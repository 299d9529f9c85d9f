# Final-state check: full GPU suite, smoke, both bench arms.
export PYTHONPATH=.
mkdir -p gpurun_out
( timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 ) > gpurun_out/final_tests.log 2>&1
( timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -5 ) > gpurun_out/final_smoke.log 2>&1
( /usr/bin/time -v timeout 1500 python bench.py 2> gpurun_out/final_bench.err | tail -1 ) > gpurun_out/final_bench.json
( timeout 600 python bench.py --impl reference 2> gpurun_out/final_bench_ref.err | tail -1 ) > gpurun_out/final_bench_ref.json
tail -3 gpurun_out/final_tests.log; cat gpurun_out/final_smoke.log; cut -c1-1500 gpurun_out/final_bench.json; grep -i "elapsed" gpurun_out/final_bench.err
