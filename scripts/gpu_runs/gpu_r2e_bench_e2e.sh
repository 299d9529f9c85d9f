# why the bench's e2e differs from scripts/time_e2e_pipe.py
export PYTHONPATH=.
timeout 300 python scripts/time_e2e_pipe.py tc_f16 "1;" 2>&1 | tail -2
for i in 1 2; do
timeout 300 python bench.py --no-outer --no-large --no-cpu-baseline > gpurun_out/be.json 2> gpurun_out/be.err; grep "e2e times" gpurun_out/be.err
python -c "
import json;d=json.load(open('gpurun_out/be.json'));print(d['e2e'])"
done
