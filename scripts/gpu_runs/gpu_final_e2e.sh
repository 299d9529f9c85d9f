export PYTHONPATH=.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max,pcie.link.width.max --format=csv
nvidia-smi topo -m 2>&1 | head -8
python - <<'PY'
import torch, time
x = torch.empty(3510000//4).pin_memory(); d = torch.empty_like(x, device='cuda')
for name, f in (("h2d", lambda: d.copy_(x, non_blocking=True)), ("d2h", lambda: x.copy_(d, non_blocking=True))):
    for _ in range(5): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50): f()
    b.record(); b.synchronize()
    ms = a.elapsed_time(b)/50
    print(name, f"{ms:.4f} ms  {3.51e6/ms/1e6:.1f} GB/s")
PY
timeout 300 python scripts/time_e2e_pipe.py tc_f16 2>&1 | tail -3
