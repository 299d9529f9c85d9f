export PYTHONPATH=.
mkdir -p gpurun_out
( timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -6 ) > gpurun_out/final_tests2.log 2>&1
tail -3 gpurun_out/final_tests2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -2
( timeout 1500 python bench.py 2> gpurun_out/final_bench3.err | tail -1 ) > gpurun_out/final_bench3.json
tail -1 gpurun_out/final_bench3.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/final_bench3.json'))
print(d['value'], d['ms_per_step'], d['e2e'], d['roofline']['frac'], d['gpu_launches'])
PY
