export PYTHONPATH=.
mkdir -p gpurun_out
S=$(date +%s)
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --comm --steps 10 --warmup 3 2> gpurun_out/final_comm.err | tail -1 > gpurun_out/final_comm.json
echo "comm bench rc=$? wall $(( $(date +%s) - S )) s"; tail -3 gpurun_out/final_comm.err; cut -c1-400 gpurun_out/final_comm.json
python - <<'PY'
import json
d=json.load(open('gpurun_out/final_comm.json'))
print(d['value'], d['e2e']['value'], d['e2e'].get('pcie_probe'), d['config'])
o=d.get('outer',{})
for k,v in o.get('c2',{}).items():
    if isinstance(v,dict) and 'ms_per_step' in v: print(k, v['ms_per_step'], v.get('iterations'))
print(o.get('c3',{}).get('ap',{}).get('ms_per_step'))
PY
