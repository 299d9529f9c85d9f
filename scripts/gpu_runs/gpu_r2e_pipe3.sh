# model-chosen row chunks: e2e timing, full GPU tests, default bench line
export PYTHONPATH=.
for r in 1 2; do for pipe in "" 1; do
  WGP_HV_PIPE=$pipe timeout 120 python scripts/time_e2e_pipe.py tc_f16 2>&1 | tail -1
done; done
timeout 120 python scripts/time_e2e_pipe.py tc 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['ms_per_step'],d['e2e'],d['roofline']['frac'],d['roofline']['kernel_ms'])"
