# round-2 final session: HEAD check -- smoke, full GPU tests, default bench line
export PYTHONPATH=.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -40 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.json
