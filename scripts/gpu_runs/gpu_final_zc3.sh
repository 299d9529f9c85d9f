export PYTHONPATH=.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_cpp_adapter.py -q -x -k "zero_copy or row_chunks or hv_ or adapter" 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -1
( timeout 1500 python bench.py 2> gpurun_out/final_bench5.err | tail -1 ) > gpurun_out/final_bench5.json
python - <<'PY'
import json
d=json.load(open('gpurun_out/final_bench5.json'))
print('value', d['value'], 'e2e', d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['pcie_probe']['h2d_GBps'], 'frac', d['roofline']['frac'])
PY
