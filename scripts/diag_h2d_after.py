"""What puts H2D into the slow state: the rate of a pinned 3.51 MB H2D copy issued
right after different GPU activities (each followed by a device synchronize)."""
import time
import torch

NB = 3510000
x = torch.empty(NB // 4).pin_memory()
d = torch.empty(NB // 4, device="cuda")
big = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
bigf = big.view(torch.float32)
small = torch.empty(8 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.Stream()


def h2d():
    with torch.cuda.stream(st):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        d.copy_(x, non_blocking=True)
        b.record(st)
        b.synchronize()
    return NB / a.elapsed_time(b) / 1e6


acts = {
    "nothing": lambda: None,
    "memset 512 MB": lambda: big.zero_(),
    "read-sum 512 MB": lambda: bigf.sum(),
    "memset 8 MB": lambda: small.zero_(),
    "memset 512 MB + 0.5 ms sleep": lambda: (big.zero_(), torch.cuda.synchronize(), time.sleep(0.0005)),
    "memset 512 MB + 5 ms sleep": lambda: (big.zero_(), torch.cuda.synchronize(), time.sleep(0.005)),
    "memset 512 MB + small H2D first": lambda: (big.zero_(), small[:4096].copy_(x.view(torch.uint8)[:4096], non_blocking=True)),
    "d2d copy 256 MB": lambda: big[: 256 << 20].copy_(big[256 << 20:]),
}
for _ in range(20):
    h2d()
for rnd in range(2):
    for name, f in acts.items():
        out = []
        for i in range(10):
            f()
            torch.cuda.synchronize()
            out.append(h2d())
        print(f"{name:34s}: " + " ".join(f"{v:5.1f}" for v in out) + " GB/s")
