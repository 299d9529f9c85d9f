export PYTHONPATH=.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -2
( timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 ) > gpurun_out/final_tests3.log 2>&1
tail -2 gpurun_out/final_tests3.log
( timeout 1500 python bench.py 2> gpurun_out/final_bench4.err | tail -1 ) > gpurun_out/final_bench4.json
( timeout 600 python bench.py --impl reference 2> gpurun_out/final_bench4_ref.err | tail -1 ) > gpurun_out/final_bench4_ref.json
python - <<'PY'
import json
d=json.load(open('gpurun_out/final_bench4.json')); r=json.load(open('gpurun_out/final_bench4_ref.json'))
print('value', d['value'], 'e2e', d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['pcie_probe'], 'frac', d['roofline']['frac'])
print('ref', r['value'], 'e2e ratio', d['e2e']['value']/r['value'], 'device ratio', d['value']/r['value'])
PY
