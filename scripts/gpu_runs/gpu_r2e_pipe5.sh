# row chunks (model) vs fixed cuts vs one launch, interleaved; full GPU tests; bench
export PYTHONPATH=.
timeout 300 python scripts/time_e2e_pipe.py tc_f16 "1;;0.68,0.32;0.72,0.28" 2>&1 | tail -4
timeout 300 python scripts/time_e2e_pipe.py tc "1;" 2>&1 | tail -2
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['ms_per_step'],d['e2e'],d['roofline']['frac'],d['roofline']['kernel_ms'])"
